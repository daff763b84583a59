"""Per-stage CUDA-event times of the batched RGB loop at config 2."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1809_06417_b200 import ReconstructionConfig, RenderConfig, _lib, render_view  # noqa: E402
from paper_1809_06417_b200.engine import ChannelLoop  # noqa: E402
from paper_1809_06417_b200.preprocess import DeviceFrames  # noqa: E402
from paper_1809_06417_b200.reconstruct import _loop_config  # noqa: E402
from paper_1809_06417_b200.synth import synth_cameras, synth_volume  # noqa: E402
from paper_1809_06417_b200.volume import compute_visual_hull  # noqa: E402

vols = synth_volume((bench.N_VOX,) * 3, seed=0, kind="flame")
truth = [vols[t] for t in ("red", "green", "blue")]
cams = synth_cameras(bench.N_VIEWS, radius=0.38, fov=60.0, elevation_jitter_deg=5.0, width=bench.RES,
                     height=bench.RES, seed=0)
rcfg = RenderConfig(tau=bench.TAU, scattering_enabled=True, sigma_s=bench.SIGMA_S, scatter_dirs=bench.SCAT_DIRS)
imgs = [render_view(c, truth, None, rcfg) for c in cams]
geom = truth[0].copy()
frames = DeviceFrames(imgs)
hull = compute_visual_hull(geom, frames.bits, cams)
b = frames.bbox
for det, nch in ((True, 3), (True, 1), (False, 3), (False, 1)):
    cfg = ReconstructionConfig(alpha_l=bench.ALPHA_L, tau=bench.TAU, max_iters=60, converge_eps=1e-12,
                               deterministic_mode=det)
    if nch == 3:
        src = frames.blanked[:, b.v0:b.v1 + 1, b.u0:b.u1 + 1, :].permute(3, 0, 1, 2).contiguous()
    else:
        src = frames.channel_crops(1)
    loop = ChannelLoop(cams, geom, None, src, frames.bits, b, hull.inside_voxels(), None, rcfg,
                       _loop_config(cfg, geom), 60, background=[0.0] * nch, use_graph=False, n_channels=nch)
    stages = [(n, f) for n, f in loop.stages() if f is not None]
    stream = _lib.stream_ptr()
    times = {n: [] for n, _ in stages}
    for it in range(25):
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(len(stages) + 1)]
        evs[0].record()
        for i, (_, fn) in enumerate(stages):
            fn(stream)
            evs[i + 1].record()
        torch.cuda.synchronize()
        if it >= 5:
            for i, (n, _) in enumerate(stages):
                times[n].append(evs[i].elapsed_time(evs[i + 1]))
    print("det" if det else "sto", nch, {n: round(float(np.mean(v)), 4) for n, v in times.items()})
    del loop
