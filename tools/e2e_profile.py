"""Phase timing of one reconstruct_channel call at the bench workload (diagnostic)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_1809_06417_b200 import ReconstructionConfig, reconstruct_channel
from paper_1809_06417_b200 import engine as eng

sc = bench.make_scene()
cfg = ReconstructionConfig(alpha_l=bench.ALPHA_L, alpha_d=1.0, tau=bench.TAU, max_iters=int(sys.argv[1]) if len(sys.argv) > 1 else 50,
                           converge_eps=1e-12, deterministic_mode=True)
orig_init = eng.ChannelLoop.__init__
orig_run = eng.ChannelLoop.run
orig_plan = eng.ChannelLoop._build_plan
orig_capture = eng.ChannelLoop.capture
times = {}


def timed(name, fn):
    def w(*a, **k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn(*a, **k)
        torch.cuda.synchronize()
        times[name] = times.get(name, 0.0) + (time.perf_counter() - t0) * 1e3
        return r
    return w


eng.ChannelLoop.__init__ = timed("init(total)", orig_init)
eng.ChannelLoop._build_plan = timed("build_plan", orig_plan)
eng.ChannelLoop.capture = timed("graph_capture", orig_capture)
eng.ChannelLoop.run = timed("run(total)", orig_run)
for rep in range(3):
    times.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    grid, trace = reconstruct_channel(sc["images"], sc["cams"], sc["geom"], sc["hull"], cfg, render_cfg=sc["rcfg"],
                                      masks=sc["masks"], bbox=sc["bbox"])
    torch.cuda.synchronize()
    total = (time.perf_counter() - t0) * 1e3
    print(f"rep {rep}: total {total:.1f} ms, iters {trace.iterations}, " + ", ".join(f"{k} {v:.1f}" for k, v in times.items()))
