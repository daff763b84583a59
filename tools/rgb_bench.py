"""reconstruct_color at BASELINE config 2 (128^3, 8 views 512^2, full RTE):
batched RGB loop vs three sequential channel loops, 50 iterations each,
wall time of the public call (median of 3).  Prints one JSON line."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1809_06417_b200 import ReconstructionConfig, RenderConfig, reconstruct_color, render_view  # noqa: E402
from paper_1809_06417_b200.synth import synth_cameras, synth_volume  # noqa: E402

vols = synth_volume((bench.N_VOX,) * 3, seed=0, kind="flame")
truth = [vols[t] for t in ("red", "green", "blue")]
cams = synth_cameras(bench.N_VIEWS, radius=0.38, fov=60.0, elevation_jitter_deg=5.0, width=bench.RES,
                     height=bench.RES, seed=0)
rcfg = RenderConfig(tau=bench.TAU, scattering_enabled=True, sigma_s=bench.SIGMA_S, scatter_dirs=bench.SCAT_DIRS)
imgs = [render_view(c, truth, None, rcfg) for c in cams]
geom = truth[0].copy()
out = {}
for det in (True, False):
    cfg = ReconstructionConfig(alpha_l=bench.ALPHA_L, alpha_d=1.0, tau=bench.TAU, max_iters=50, converge_eps=1e-12,
                               deterministic_mode=det)
    for mode in ("1", "0"):
        os.environ["FVR_RGB_BATCH"] = mode
        reconstruct_color(imgs, cams, geom, cfg, render_cfg=rcfg)  # warm
        walls = []
        for _ in range(3):
            t0 = time.perf_counter()
            res = reconstruct_color(imgs, cams, geom, cfg, render_cfg=rcfg)
            walls.append(time.perf_counter() - t0)
        its = min(tr.iterations for tr in res.traces.values())
        key = ("deterministic" if det else "stochastic") + ("_batched" if mode == "1" else "_sequential")
        out[key] = {"rgb_iters_per_s": its / float(np.median(walls)), "calls_ms": [1e3 * w for w in walls],
                    "iterations": its}
print(json.dumps({"workload": "reconstruct_color, config 2 (128^3, 8 views 512^2, sigma_s 0.1, 32 dirs), "
                              "50 iterations per channel, public API with host images", **out}))
