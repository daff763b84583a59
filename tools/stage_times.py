"""Per-stage device time of the loop at one BASELINE config (events between
the stages, 5 iterations after 3 warm-up ones), plus the plan sizes:
  python tools/stage_times.py 4"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_1809_06417_b200 import ReconstructionConfig, _lib  # noqa: E402
from paper_1809_06417_b200.engine import ChannelLoop  # noqa: E402
from paper_1809_06417_b200.reconstruct import _init_grid, _loop_config  # noqa: E402

torch.cuda.set_device(0)
cfg_no = int(sys.argv[1]) if len(sys.argv) > 1 else 2
sc = workloads.device_scene(*workloads.CONFIGS[cfg_no])
cfg = ReconstructionConfig(alpha_l=0.006, alpha_d=1.0, tau=sc["tau"], max_iters=20, converge_eps=1e-12,
                           deterministic_mode=os.environ.get("STAGE_STOCHASTIC") != "1", g_sigma=0.1, rng_seed=0)
grid0 = _init_grid(sc["geom"], sc["hull"], "green")
src = [im.data[sc["bbox"].slices][:, :, 0] for im in sc["images"]]
loop = ChannelLoop(sc["cams"], grid0, grid0.values, src, sc["masks"], sc["bbox"], sc["hull"].inside_voxels(),
                   sc["hull"].key_point_mask(), sc["rcfg"], _loop_config(cfg, grid0), 20, use_graph=False)
stages = [(n, f) for n, f in loop.stages() if f is not None]
stream = _lib.stream_ptr()
for _ in range(3):
    for _, f in stages:
        f(stream)
evs = []
for _ in range(5):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(len(stages) + 1)]
    e[0].record()
    for i, (_, f) in enumerate(stages):
        f(stream)
        e[i + 1].record()
    evs.append(e)
torch.cuda.synchronize()
ms = {n: float(np.mean([e[i].elapsed_time(e[i + 1]) for e in evs])) for i, (n, _) in enumerate(stages)}
row_b = (0 if loop._static_zero else 8) + (8 if any(b != 0.0 for b in loop.background) else 0)  # base, t_fin
rb = 6 * loop.rplan_nnz + row_b * loop.rp_len.numel() * 32 + 8 * sum(s.size for s in src)
ab = 6 * loop.plan_slots + 20 * loop.n_kp
print(json.dumps({"config": cfg_no, "stage_ms": ms, "render_gb": rb / 1e9, "adjust_gb": ab / 1e9,
                  "render_tbs": rb / ms.get("render", 1e9) / 1e9, "adjust_tbs": ab / ms.get("adjust", 1e9) / 1e9,
                  "n_kp": loop.n_kp, "adj_wide": bool(getattr(loop, "adj_wide", False)),
                  "rp_wide": bool(getattr(loop, "rp_wide", False))}))
