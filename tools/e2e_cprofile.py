"""cProfile of one steady-state reconstruct_channel call at the bench workload (diagnostic)."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_1809_06417_b200 import ReconstructionConfig, reconstruct_channel

sc = bench.make_scene()
cfg = ReconstructionConfig(alpha_l=bench.ALPHA_L, alpha_d=1.0, tau=bench.TAU, max_iters=50, converge_eps=1e-12,
                           deterministic_mode=True)
args = (sc["images"], sc["cams"], sc["geom"], sc["hull"], cfg)
kw = dict(render_cfg=sc["rcfg"], masks=sc["masks"], bbox=sc["bbox"])
for _ in range(2):
    reconstruct_channel(*args, **kw)
torch.cuda.synchronize()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
reconstruct_channel(*args, **kw)
torch.cuda.synchronize()
pr.disable()
print(f"total {(time.perf_counter() - t0) * 1e3:.1f} ms")
pstats.Stats(pr).sort_stats("tottime").print_stats(30)
pstats.Stats(pr).sort_stats("cumulative").print_stats(30)
