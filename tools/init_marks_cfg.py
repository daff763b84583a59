"""Host / device timeline of ChannelLoop setup at one BASELINE config
(FVR_INIT_PROFILE marks), second construction (warm):
  python tools/init_marks_cfg.py 4"""
import os
import sys

os.environ["FVR_INIT_PROFILE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_1809_06417_b200 import ReconstructionConfig  # noqa: E402
from paper_1809_06417_b200.engine import ChannelLoop  # noqa: E402
from paper_1809_06417_b200.reconstruct import _init_grid, _loop_config  # noqa: E402

torch.cuda.set_device(0)
cfg_no = int(sys.argv[1]) if len(sys.argv) > 1 else 4
sc = workloads.device_scene(*workloads.CONFIGS[cfg_no])
cfg = ReconstructionConfig(alpha_l=0.006, alpha_d=1.0, tau=sc["tau"], max_iters=5, converge_eps=1e-12,
                           deterministic_mode=True)
src = [im.data[sc["bbox"].slices][:, :, 0] for im in sc["images"]]
inside = sc["hull"].inside_voxels()
for rep in range(2):
    torch.cuda.synchronize()
    loop = ChannelLoop(sc["cams"], sc["geom"], None, src, sc["masks"], sc["bbox"], inside, None, sc["rcfg"],
                       _loop_config(cfg, sc["geom"]), 5, use_graph=False)
    m = loop._marks
    torch.cuda.synchronize()
    if rep:
        t0 = m[0][1]
        for (name, th, ev), prev in zip(m[1:], m):
            print(f"  {name:24s} host {1e3 * (th - t0):8.3f} ms (+{1e3 * (th - prev[1]):7.3f})  "
                  f"device +{prev[2].elapsed_time(ev):8.3f} ms")
    del loop
    torch.cuda.empty_cache()
