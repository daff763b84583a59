"""Is a reconstruct_channel call's ChannelLoop freed when the call returns
(refcount), or only by the cyclic GC later (its plan buffers then stay
allocated into the next call, which must cudaMalloc fresh ones)?"""
import gc
import sys
import time
import weakref

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1809_06417_b200 import ReconstructionConfig, reconstruct_channel  # noqa: E402
from paper_1809_06417_b200 import engine  # noqa: E402

sc = bench.make_scene()
import os  # noqa: E402

cfg = ReconstructionConfig(alpha_l=bench.ALPHA_L, alpha_d=1.0, tau=bench.TAU, max_iters=50, converge_eps=1e-12,
                           deterministic_mode=os.environ.get("E2E_STOCHASTIC") != "1", g_sigma=0.1, rng_seed=0)
refs = []
orig_init = engine.ChannelLoop.__init__


def init(self, *a, **k):
    orig_init(self, *a, **k)
    refs.append(weakref.ref(self))


engine.ChannelLoop.__init__ = init
for i in range(8):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    reconstruct_channel(sc["images"], sc["cams"], sc["geom"], sc["hull"], cfg, render_cfg=sc["rcfg"],
                        masks=sc["masks"], bbox=sc["bbox"])
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) * 1e3
    alive = sum(r() is not None for r in refs)
    print(f"call {i}: {dt:.2f} ms, loops alive after return: {alive}, reserved {torch.cuda.memory_reserved() / 1e9:.2f} GB")
    if alive:
        obj = [r() for r in refs if r() is not None][0]
        for ref in gc.get_referrers(obj)[:6]:
            print("   referrer:", type(ref), str(ref)[:150])
        del obj
