"""Per-phase wall time of repeated reconstruct_channel calls (variance hunt)."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1809_06417_b200 import ReconstructionConfig, reconstruct_channel  # noqa: E402
from paper_1809_06417_b200 import engine  # noqa: E402

sc = bench.make_scene()
cfg = ReconstructionConfig(alpha_l=bench.ALPHA_L, alpha_d=1.0, tau=bench.TAU, max_iters=50, converge_eps=1e-12,
                           deterministic_mode=True)
orig_init, orig_run = engine.ChannelLoop.__init__, engine.ChannelLoop.run
ph = {}


def init(self, *a, **k):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    orig_init(self, *a, **k)
    torch.cuda.synchronize()
    ph["init"] = (time.perf_counter() - t0) * 1e3


def run(self, *a, **k):
    t0 = time.perf_counter()
    r = orig_run(self, *a, **k)
    ph["run"] = (time.perf_counter() - t0) * 1e3
    return r


engine.ChannelLoop.__init__, engine.ChannelLoop.run = init, run
for i in range(8):
    t0 = time.perf_counter()
    reconstruct_channel(sc["images"], sc["cams"], sc["geom"], sc["hull"], cfg, render_cfg=sc["rcfg"],
                        masks=sc["masks"], bbox=sc["bbox"])
    tot = (time.perf_counter() - t0) * 1e3
    print(f"call {i}: total {tot:6.1f} ms  init {ph['init']:6.1f}  run {ph['run']:6.1f}  other {tot - ph['init'] - ph['run']:6.1f}")
