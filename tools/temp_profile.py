"""Where a config-3 reconstruct_temperature call (10 iterations) spends its
wall time: cProfile of one warm call, top entries by cumulative time."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_1809_06417_b200 import build_color_temp_map, reconstruct_temperature  # noqa: E402
from tests.fullsize_common import loop_cfg  # noqa: E402

torch.cuda.set_device(0)
sc = workloads.device_scene(*workloads.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 3])
cmap = build_color_temp_map()
cfg = loop_cfg(sc, 10)
for _ in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    reconstruct_temperature(sc["rgb"], sc["cams"], cmap, sc["geom"], cfg, render_cfg=sc["rcfg"])
    torch.cuda.synchronize()
    print(f"call {1e3 * (time.perf_counter() - t0):.1f} ms")
pr = cProfile.Profile()
pr.enable()
reconstruct_temperature(sc["rgb"], sc["cams"], cmap, sc["geom"], cfg, render_cfg=sc["rcfg"])
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(35)
