"""Where ChannelLoop.__init__ spends its time across repeated calls."""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1809_06417_b200 import ReconstructionConfig, reconstruct_channel  # noqa: E402

sc = bench.make_scene()
cfg = ReconstructionConfig(alpha_l=bench.ALPHA_L, alpha_d=1.0, tau=bench.TAU, max_iters=50, converge_eps=1e-12,
                           deterministic_mode=True)
pr = cProfile.Profile()
for i in range(8):
    if i >= 2:
        pr.enable()
    reconstruct_channel(sc["images"], sc["cams"], sc["geom"], sc["hull"], cfg, render_cfg=sc["rcfg"],
                        masks=sc["masks"], bbox=sc["bbox"])
    if i >= 2:
        pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
print(torch.cuda.memory_stats()["num_alloc_retries"], torch.cuda.memory_stats()["segment.all.allocated"],
      torch.cuda.memory_stats()["segment.all.freed"])
