"""reconstruct_channel at config 2 (50 iterations) with and without a
per-iteration snapshot callback: the snapshot ring keeps the loop on the
device (§8f rank 4)."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1809_06417_b200 import ReconstructionConfig, reconstruct_channel  # noqa: E402

sc = bench.make_scene()
cfg = ReconstructionConfig(alpha_l=bench.ALPHA_L, alpha_d=1.0, tau=bench.TAU, max_iters=50, converge_eps=1e-12,
                           deterministic_mode=True)
out = {}
for name, cb in (("no_callback", None), ("snapshot_callback", lambda it, g, r: None)):
    reconstruct_channel(sc["images"], sc["cams"], sc["geom"], sc["hull"], cfg, render_cfg=sc["rcfg"],
                        masks=sc["masks"], bbox=sc["bbox"], callback=cb)
    walls = []
    for _ in range(3):
        t0 = time.perf_counter()
        reconstruct_channel(sc["images"], sc["cams"], sc["geom"], sc["hull"], cfg, render_cfg=sc["rcfg"],
                            masks=sc["masks"], bbox=sc["bbox"], callback=cb)
        walls.append(time.perf_counter() - t0)
    out[name] = {"iters_per_s": 50 / float(np.median(walls)), "calls_ms": [1e3 * w for w in walls]}
print(json.dumps(out))
