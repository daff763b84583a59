"""Host timeline of ChannelLoop setup (FVR_INIT_PROFILE marks): host ms since
the loop's start at each mark and the device time between marks."""
import os
import sys

os.environ["FVR_INIT_PROFILE"] = "1"
sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1809_06417_b200 import ReconstructionConfig, reconstruct_channel  # noqa: E402
from paper_1809_06417_b200 import engine  # noqa: E402

sc = bench.make_scene()
cfg = ReconstructionConfig(alpha_l=bench.ALPHA_L, alpha_d=1.0, tau=bench.TAU, max_iters=50,
                           converge_eps=1e-12, deterministic_mode=os.environ.get("E2E_STOCHASTIC") != "1", g_sigma=0.1, rng_seed=0)
loops = []
orig = engine.ChannelLoop.__init__


def init(self, *a, **k):
    orig(self, *a, **k)
    loops.append(self)


engine.ChannelLoop.__init__ = init
for i in range(5):
    reconstruct_channel(sc["images"], sc["cams"], sc["geom"], sc["hull"], cfg, render_cfg=sc["rcfg"],
                        masks=sc["masks"], bbox=sc["bbox"])
    loop = loops.pop()
    if i >= 3:
        m = loop._marks
        t0 = m[0][1]
        for (name, th, ev), prev in zip(m[1:], m):
            print(f"  {name:24s} host {1e3 * (th - t0):6.3f} ms (+{1e3 * (th - prev[1]):5.3f})  "
                  f"device +{prev[2].elapsed_time(ev):6.3f} ms")
        print()
    del loop
