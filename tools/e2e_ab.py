"""Interleaved A/B of the public reconstruct_channel call (config 2, 50
iterations) under setup variants, in one process so box-to-box variance
cancels: python tools/e2e_ab.py [rounds]

Variants: "base" (defaults), "sync_sizes" (the plan sizes read by a
pageable .cpu() at the point of use, the pre-HostRead behaviour); add
variants to ``setup`` (environment switches are read per call).

Measured (config 2, 15 rounds): base 10.241 ms, sync_sizes 10.227 ms, and an
adjust count pass queued after the render fill 10.265 ms -- the setup is
device-bound, host-side reordering moves nothing."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1809_06417_b200 import ReconstructionConfig, _lib, reconstruct_channel  # noqa: E402

sc = bench.make_scene()
cfg = ReconstructionConfig(alpha_l=bench.ALPHA_L, alpha_d=1.0, tau=bench.TAU, max_iters=50, converge_eps=1e-12,
                           deterministic_mode=os.environ.get("E2E_STOCHASTIC") != "1", g_sigma=0.1, rng_seed=0)
HostRead = _lib.HostRead


class SyncRead:
    def __init__(self, tensor):
        self.tensor = tensor

    def get(self):
        return self.tensor.cpu().tolist()


def setup(name):
    _lib.HostRead = SyncRead if name == "sync_sizes" else HostRead
    if name == "no_row_sort":
        os.environ["FVR_SPLAN_SORT"] = "0"
    else:
        os.environ.pop("FVR_SPLAN_SORT", None)
    if name == "clear_first":
        os.environ["FVR_PAD_ZERO"] = "0"
    else:
        os.environ.pop("FVR_PAD_ZERO", None)
    if name == "side_prio0":
        os.environ["FVR_SIDE_PRIORITY"] = "0"
    else:
        os.environ.pop("FVR_SIDE_PRIORITY", None)
    if name in ("fill_overlap", "fill_serial"):
        os.environ["FVR_FILL_SERIAL"] = "0" if name == "fill_overlap" else "1"
    else:
        os.environ.pop("FVR_FILL_SERIAL", None)


def call():
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    reconstruct_channel(sc["images"], sc["cams"], sc["geom"], sc["hull"], cfg, render_cfg=sc["rcfg"],
                        masks=sc["masks"], bbox=sc["bbox"])
    return (time.perf_counter() - t0) * 1e3


names = sys.argv[2].split(",") if len(sys.argv) > 2 else ["base", "sync_sizes"]
rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 12
for n in names:  # warm each variant
    setup(n)
    call()
    call()
res = {n: [] for n in names}
for _ in range(rounds):
    for n in names:
        setup(n)
        res[n].append(call())
for n in names:
    print(f"{n:12s} median {statistics.median(res[n]):7.3f} ms  min {min(res[n]):7.3f}  "
          f"({50e3 / statistics.median(res[n]):.0f} it/s)")
