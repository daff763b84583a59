"""Where one public-API reconstruct_channel call (config 2, 50 iterations)
spends its time: host wall clock of the phases, and device time of the loop
(CUDA events around ChannelLoop.run, excluding the result copy)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1809_06417_b200 import ReconstructionConfig, reconstruct_channel  # noqa: E402
from paper_1809_06417_b200 import engine  # noqa: E402

torch.cuda.set_device(0)
sc = bench.make_scene()
cfg = ReconstructionConfig(alpha_l=bench.ALPHA_L, alpha_d=1.0, tau=bench.TAU, max_iters=50, converge_eps=1e-12,
                           deterministic_mode=os.environ.get("E2E_STOCHASTIC") != "1", g_sigma=0.1, rng_seed=0)
rec = {}
orig_run, orig_init = engine.ChannelLoop.run, engine.ChannelLoop.__init__


def run(self, *a, **k):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    out = orig_run(self, *a, **k)
    e1.record()
    torch.cuda.synchronize()
    rec["run_host_ms"] = (time.perf_counter() - t0) * 1e3
    rec["run_device_ms"] = e0.elapsed_time(e1)
    return out


def init(self, *a, **k):
    t0 = time.perf_counter()
    orig_init(self, *a, **k)
    rec["init_host_ms"] = (time.perf_counter() - t0) * 1e3


engine.ChannelLoop.run, engine.ChannelLoop.__init__ = run, init
for chunk in (8, 16, 50):
    orig_run.__defaults__ = (None, chunk, None)
    for i in range(6):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        reconstruct_channel(sc["images"], sc["cams"], sc["geom"], sc["hull"], cfg, render_cfg=sc["rcfg"],
                            masks=sc["masks"], bbox=sc["bbox"])
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) * 1e3
        if i >= 2:
            print(f"chunk {chunk}: wall {wall:.2f} ms  init(host) {rec['init_host_ms']:.2f}  run host "
                  f"{rec['run_host_ms']:.2f} / device {rec['run_device_ms']:.2f} ms "
                  f"({rec['run_device_ms'] / 50 * 1e3:.1f} us/iter)", flush=True)
