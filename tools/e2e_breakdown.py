"""Where the e2e (public-API) time of reconstruct_channel goes at config 2:
cProfile of one warmed call, top functions by cumulative time."""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1809_06417_b200 import ReconstructionConfig, reconstruct_channel  # noqa: E402

sc = bench.make_scene()
cfg = ReconstructionConfig(alpha_l=bench.ALPHA_L, alpha_d=1.0, tau=bench.TAU, max_iters=50,
                           converge_eps=1e-12, deterministic_mode=True)


def call():
    return reconstruct_channel(sc["images"], sc["cams"], sc["geom"], sc["hull"], cfg, render_cfg=sc["rcfg"],
                               masks=sc["masks"], bbox=sc["bbox"])


call()
for _ in range(3):
    t0 = time.perf_counter()
    _, tr = call()
    print(f"wall {1e3 * (time.perf_counter() - t0):.2f} ms for {tr.iterations} iterations")
pr = cProfile.Profile()
pr.enable()
call()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(35)
