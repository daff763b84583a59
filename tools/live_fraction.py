"""How many render samples are live under the static (hull) occupancy vs the
dynamic one (values > 0) after N iterations of the bench workload (diagnostic)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_1809_06417_b200 import ReconstructionConfig, _lib
from paper_1809_06417_b200.engine import ChannelLoop
from paper_1809_06417_b200.reconstruct import _init_grid, _loop_config

sc = bench.make_scene()
cfg = ReconstructionConfig(alpha_l=bench.ALPHA_L, alpha_d=1.0, tau=bench.TAU, max_iters=60, converge_eps=1e-12,
                           deterministic_mode=True)
grid0 = _init_grid(sc["geom"], sc["hull"], "green")
src = [im.data[sc["bbox"].slices][:, :, 0] for im in sc["images"]]
loop = ChannelLoop(sc["cams"], grid0, grid0.values, src, sc["masks"], sc["bbox"], sc["hull"].inside_voxels(),
                   sc["hull"].key_point_mask(), sc["rcfg"], _loop_config(cfg, grid0), cfg.max_iters,
                   background=0.0, use_graph=False)
print("static live", bench.live_samples(sc, loop.occ))
dyn = torch.empty_like(loop.occ)
for it in (1, 5, 20, 50):
    while loop.read_state()["it"] < it:
        loop.launch_iteration()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _lib.call("fvr_occupancy", loop.values.data_ptr(), 1, None, loop.grid, dyn.data_ptr(), _lib.stream_ptr())
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) * 1e3
    print(f"after {it} iters: dynamic live {bench.live_samples(sc, dyn)}  (distance map {dt:.3f} ms host-timed)")
