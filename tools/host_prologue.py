"""Host time of a public reconstruct_channel call's prologue at config 2:
the staging pass and the work before ChannelLoop (medians of 20)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1809_06417_b200 import reconstruct as R  # noqa: E402

sc = bench.make_scene()
imgs, masks, bbox, hull = sc["images"], sc["masks"], sc["bbox"], sc["hull"]
for _ in range(3):
    R._stage_host_inputs(imgs, masks, bbox, hull)
torch.cuda.synchronize()
ts = []
for _ in range(20):
    t0 = time.perf_counter()
    R._stage_host_inputs(imgs, masks, bbox, hull)
    ts.append(time.perf_counter() - t0)
    torch.cuda.synchronize()
print(f"_stage_host_inputs host {1e3 * np.median(ts):.3f} ms")
from paper_1809_06417_b200 import _lib  # noqa: E402

ts = []
for _ in range(20):
    t0 = time.perf_counter()
    _lib.cameras_tensor(sc["cams"], _lib.device())
    ts.append(time.perf_counter() - t0)
print(f"cameras_tensor host {1e3 * np.median(ts):.3f} ms")
