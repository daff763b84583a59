"""Render-plan padding at config 2: stored SELL slots vs entries with a
non-zero weight, and the per-unit spread of row lengths."""
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1809_06417_b200 import ReconstructionConfig, _lib  # noqa: E402
from paper_1809_06417_b200.engine import ChannelLoop  # noqa: E402
from paper_1809_06417_b200.reconstruct import _init_grid, _loop_config  # noqa: E402

t = _lib.torch()
sc = bench.make_scene()
cfg = ReconstructionConfig(alpha_l=bench.ALPHA_L, alpha_d=1.0, tau=bench.TAU, max_iters=10, converge_eps=1e-12)
grid0 = _init_grid(sc["geom"], sc["hull"], "green")
src = [im.data[sc["bbox"].slices][:, :, 0] for im in sc["images"]]
loop = ChannelLoop(sc["cams"], grid0, grid0.values, src, sc["masks"], sc["bbox"], sc["hull"].inside_voxels(),
                   sc["hull"].key_point_mask(), sc["rcfg"], _loop_config(cfg, grid0), 10, use_graph=False)
a = loop.rp_a
nz = (a != 0)  # exponent bits in the top byte: zero only for a zero weight (index 0)
slots = a.shape[0]
print("slots", slots, "nonzero", int(nz.sum()), "fill", float(nz.sum()) / slots)
n_units = loop.rp_len.numel()
rowlen = t.zeros(n_units * 32, dtype=t.int64, device=e.device)
# a word of entry t of row (unit, lane) at unit_off[unit]*32 + 128 (t // 4) + 4 lane + t % 4
off = loop.rp_off[:-1]
unit_of_slot = t.repeat_interleave(t.arange(n_units, device=e.device), loop.rp_len.long() * 32)
lane = ((t.arange(slots, device=e.device) - off[unit_of_slot] * 32) % 128) // 4
rowlen.index_add_(0, unit_of_slot * 32 + lane, nz.long())
rl = rowlen.view(n_units, 32).float()
mx = rl.max(1).values
print("units", n_units, "mean row", float(rl.mean()), "mean unit max", float(mx.mean()),
      "max unit", float(mx.max()))

# padding if the 32 pixels of a unit were the length-sorted pixels of a larger
# tile (SELL-C-sigma style, sigma = tile pixels)
upv = loop.bpv
V = n_units // upv
ux = (loop.w_bb + 7) // 8
uy = upv // ux
img = rl.view(V, uy, ux, 4, 8).permute(0, 1, 3, 2, 4).reshape(V, uy * 4, ux * 8)
for th, tw in [(4, 8), (8, 8), (4, 16), (8, 16), (16, 16), (16, 32), (32, 32)]:
    H, W = (uy * 4) // th * th, (ux * 8) // tw * tw
    tiles = img[:, :H, :W].reshape(V, H // th, th, W // tw, tw).permute(0, 1, 3, 2, 4).reshape(-1, th * tw)
    srt = tiles.sort(1, descending=True).values.view(tiles.shape[0], -1, 32)
    print(f"tile {th}x{tw}: padded slots / nonzero = {float(srt.max(2).values.sum() * 32) / float(tiles.sum()):.4f}")
