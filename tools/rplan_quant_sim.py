"""Precision of candidate render-plan weight formats (diagnostic): builds the
config-2 render plan with f32 weights (FVR_WIDE_PLANS=1), then evaluates
rec = B c with c = max(truth, 0) at the hull key points for
  f32      the exact weights,
  m17      the current 6-byte format (exponent + 16 stored mantissa bits),
  c8q16    16-bit fixed point with one exponent per 8-entry lane chunk,
  r16      16-bit fixed point with one exponent per row,
and prints the max and rms error relative to max(|rec|, 1)."""
import os
import sys

os.environ["FVR_WIDE_PLANS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_1809_06417_b200 import ReconstructionConfig  # noqa: E402
from paper_1809_06417_b200.engine import ChannelLoop  # noqa: E402
from paper_1809_06417_b200.reconstruct import _init_grid, _loop_config  # noqa: E402

torch.cuda.set_device(0)
sc = workloads.device_scene(*workloads.CONFIGS[2])
cfg = ReconstructionConfig(alpha_l=0.006, alpha_d=1.0, tau=sc["tau"], max_iters=3, converge_eps=1e-12,
                           deterministic_mode=True)
grid0 = _init_grid(sc["geom"], sc["hull"], "green")
src = [im.data[sc["bbox"].slices][:, :, 0] for im in sc["images"]]
loop = ChannelLoop(sc["cams"], grid0, grid0.values, src, sc["masks"], sc["bbox"], sc["hull"].inside_voxels(),
                   sc["hull"].key_point_mask(), sc["rcfg"], _loop_config(cfg, grid0), 3, use_graph=False)
assert loop.rplan and loop.rp_wide
A = loop.rp_a.cpu().numpy().view(np.uint32)
W = loop.rp_b.cpu().numpy().view(np.float32)
off = loop.rp_off.cpu().numpy()
n_units = off.size - 1
truth = np.maximum(sc["truth"][1].values.reshape(-1), 0)
kp = loop.kp[: loop.n_kp].cpu().numpy()
c = truth[kp].astype(np.float64)
K = 8  # entries per lane chunk (wide: kRpA)
# entry (unit u, lane l, t) at ((off[u] / K + t / K) * 32 + l) * K + t % K
rows = []
errs = {k: [] for k in ("m17", "c8q16", "r16")}
ref_all = []
lens = np.diff(off)
rng = np.random.default_rng(0)
units = rng.choice(n_units, size=min(n_units, 3000), replace=False)


def m17(w):
    b = w.view(np.uint32)
    b = ((b + 0x40) >> 7) << 7
    return b.view(np.float32).astype(np.float64)


def q16(w, wmax):
    e = np.ceil(np.log2(np.maximum(wmax, 1e-38)))  # 2^e >= wmax
    s = 2.0 ** (e - 16)
    return np.round(w / s) * s


for u in units:
    L = lens[u]
    if L == 0:
        continue
    t = np.arange(L)
    for lane in range(32):
        idx = ((off[u] // K + t // K) * 32 + lane) * K + t % K
        col = A[idx].astype(np.int64)
        w = W[idx]
        ref = float(np.dot(w.astype(np.float64), c[col]))
        ref_all.append(ref)
        den = max(abs(ref), 1.0)
        errs["m17"].append(abs(np.dot(m17(w), c[col]) - ref) / den)
        wc = w.reshape(-1, K).astype(np.float64)
        cm = wc.max(1, keepdims=True)
        errs["c8q16"].append(abs(np.dot(q16(wc, cm).reshape(-1), c[col]) - ref) / den)
        errs["r16"].append(abs(np.dot(q16(w.astype(np.float64), w.max()), c[col]) - ref) / den)
print("rows", len(ref_all), "max |rec|", max(ref_all))
for k, v in errs.items():
    v = np.array(v)
    print(f"{k:6s} max {v.max():.3e}  rms {np.sqrt((v ** 2).mean()):.3e}")
