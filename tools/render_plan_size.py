"""Diagnostic: size of a fixed forward-render operator B (rows = bbox pixels,
columns = hull key points) at config 2 -- distinct (pixel, key point) pairs
over the 3x3x3 stencils of every live sample, counted with torch."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1809_06417_b200.engine import ChannelLoop  # noqa: E402
from paper_1809_06417_b200.geometry import pixel_rays  # noqa: E402
from paper_1809_06417_b200.reconstruct import _init_grid, _loop_config  # noqa: E402
from paper_1809_06417_b200 import ReconstructionConfig  # noqa: E402

sc = bench.make_scene()
geom, bbox = sc["geom"], sc["bbox"]
cfg = ReconstructionConfig(alpha_l=bench.ALPHA_L, tau=bench.TAU, max_iters=2, deterministic_mode=True)
grid0 = _init_grid(geom, sc["hull"], "green")
src = [im.data[bbox.slices][:, :, 0] for im in sc["images"]]
loop = ChannelLoop(sc["cams"], grid0, grid0.values, src, sc["masks"], bbox, sc["hull"].inside_voxels(),
                   sc["hull"].key_point_mask(), sc["rcfg"], _loop_config(cfg, grid0), 2, use_graph=False)
dev = loop.occ.device
occ = loop.occ.reshape(-1)
hullkp = torch.from_numpy(sc["hull"].key_point_mask().reshape(-1)).to(dev)
lo = torch.tensor(geom.origin, dtype=torch.float64, device=dev)
n = torch.tensor([geom.nx, geom.ny, geom.nz], dtype=torch.float64, device=dev)
hi = lo + n * geom.edge
sx, sy = (geom.ny + 1) * (geom.nz + 1), geom.nz + 1
offs = torch.tensor([dx * sx + dy * sy + dz for dx in (-1, 0, 1) for dy in (-1, 0, 1) for dz in (-1, 0, 1)],
                    device=dev)
us = np.arange(bbox.u0, bbox.u1 + 1) + 0.5
vs = np.arange(bbox.v0, bbox.v1 + 1) + 0.5
uu, vv = np.meshgrid(us, vs, indexing="xy")
pairs = live = 0
for cam in sc["cams"]:
    o_np, d_np = pixel_rays(cam, uu.ravel(), vv.ravel())
    o = torch.tensor(o_np, dtype=torch.float64, device=dev)
    for chunk in np.array_split(np.arange(d_np.shape[0]), 16):
        d = torch.tensor(d_np[chunk], dtype=torch.float64, device=dev)
        t0 = (lo - o) / d
        t1 = (hi - o) / d
        tmin = torch.where(d == 0, torch.full_like(d, -1e300), torch.minimum(t0, t1)).amax(1)
        tmax = torch.where(d == 0, torch.full_like(d, 1e300), torch.maximum(t0, t1)).amin(1)
        te = tmin.clamp(min=0.0)
        cnt = torch.where(tmax > te, torch.floor((tmax - te) / geom.edge + 1e-9), torch.zeros_like(te)).long()
        kmax = int(cnt.max().item())
        if kmax == 0:
            continue
        qb = ((o - lo)[None, :] + (te - 0.5 * geom.edge)[:, None] * d) / geom.edge
        k = torch.arange(1, kmax + 1, dtype=torch.float64, device=dev)
        q = qb[:, None, :] + k[None, :, None] * d[:, None, :]
        m = torch.minimum(torch.clamp(torch.round(q).long(), min=0), n.long())
        idx = m[..., 0] * sx + m[..., 1] * sy + m[..., 2]
        valid = (k[None, :] <= cnt[:, None]) & (occ[idx.clamp(max=occ.numel() - 1)] <= 1)
        live += int(valid.sum())
        ray = torch.arange(idx.shape[0], device=dev)[:, None].expand_as(idx)
        kp = (idx[valid][:, None] + offs[None, :]).clamp(0, occ.numel() - 1)
        r = ray[valid][:, None].expand_as(kp)
        keep = hullkp[kp]
        key = torch.unique(r[keep] * (1 << 23) + kp[keep])
        pairs += int(key.numel())
print({"live_samples": live, "distinct_pixel_hullkp_pairs": pairs, "per_live_sample": pairs / max(live, 1),
       "bytes_at_8B": pairs * 8})
