import faulthandler, sys, os
faulthandler.enable()
sys.path.insert(0, os.getcwd())
import numpy as np
print("step0", flush=True)
from paper_1809_06417_b200 import _lib
L = _lib.load()
print("loaded", L.fvr_abi_version(), flush=True)
import torch
print("torch", torch.cuda.is_available(), flush=True)
from tests.conftest import load_golden
k = load_golden("kernels.npz")
from paper_1809_06417_b200 import _kernels
out = np.empty((k["dirs"].shape[0], 2))
_kernels.render_rays(k["origin"], k["dirs"], k["values"], k["lo"], float(k["edge"]), 0.05, 1.0, k["background"], False, 0.0, np.zeros((1,3)), 0.0, float(k["edge"]), out)
print("render_rays_host ok", np.abs(out - k["render_plain"]).max(), flush=True)
dev = torch.device("cuda", 0)
t = torch.zeros(4, device=dev)
print("torch alloc ok", flush=True)
from paper_1809_06417_b200 import build_color_temp_map
cm = build_color_temp_map()
print("ctmap ok", cm.entries.max(), flush=True)
