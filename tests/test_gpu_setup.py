"""The loop-setup index kernels (csrc/fvr_setup.cu) against plain tensor-op
restatements of the orders they produce: Morton keys of the hull key
points, the adjust plans' windowed SELL row order and the render plan's tile
row order.  The orders only decide layouts (every plan sum is order-free), but
they must be permutations with the stated sort keys."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _morton_ref(k, shape):
    sy, sx = shape[2], shape[1] * shape[2]
    x, y, z = k // sx, (k // sy) % shape[1], k % sy

    def spread(v):
        out = np.zeros_like(v)
        for b in range(21):
            out |= ((v >> b) & 1) << (3 * b)
        return out

    return (spread(x) << 2) | (spread(y) << 1) | spread(z)


def test_morton_keys(cuda_device):
    import torch

    from paper_1809_06417_b200 import _lib
    from paper_1809_06417_b200.engine import _morton_order

    rng = np.random.default_rng(0)
    for shape in ((129, 129, 129), (33, 70, 17), (513, 513, 513)):
        n = int(np.prod(shape))
        kp = np.sort(rng.choice(n, size=min(n, 200_000), replace=False)).astype(np.int32)
        d = torch.from_numpy(kp).to(cuda_device)
        keys = torch.empty(kp.size, dtype=torch.int64, device=cuda_device)
        g = _lib.FvrGrid()
        g.nx, g.ny, g.nz = shape[0] - 1, shape[1] - 1, shape[2] - 1
        g.edge = 1.0
        _lib.call("fvr_morton_keys", d.data_ptr(), kp.size, g, keys.data_ptr(), _lib.stream_ptr())
        want = _morton_ref(kp.astype(np.int64), shape)
        assert np.array_equal(keys.cpu().numpy(), want)
        ordered = _morton_order(d, shape).cpu().numpy()
        assert np.array_equal(ordered, kp[np.argsort(want, kind="stable")])


@pytest.mark.parametrize("window", [32, 128, 1024])
def test_sell_window_order(cuda_device, window):
    import torch

    from paper_1809_06417_b200 import _lib

    rng = np.random.default_rng(window)
    n = 100_003
    counts = rng.integers(0, 40, n).astype(np.int32)
    d = torch.from_numpy(counts).to(cuda_device)
    out = torch.empty(n, dtype=torch.int32, device=cuda_device)
    _lib.call("fvr_sell_window_order", d.data_ptr(), n, window, out.data_ptr(), _lib.stream_ptr())
    pos = np.arange(n)
    want = np.lexsort((pos, -counts.astype(np.int64), pos // window))  # window, longest first, row order
    assert np.array_equal(out.cpu().numpy(), want)


@pytest.mark.parametrize("tile", [(2, 4), (1, 1), (4, 8)])
def test_rplan_tile_rows(cuda_device, tile):
    import torch

    from paper_1809_06417_b200 import _lib

    rng = np.random.default_rng(tile[0] * 10 + tile[1])
    n_views, w, h = 3, 139, 255
    ux, uy = (w + 7) // 8, (h + 3) // 4
    n_units = n_views * ux * uy
    row_len = rng.integers(0, 700, n_units * 32).astype(np.int32)
    d = torch.from_numpy(row_len).to(cuda_device)
    row_src = torch.empty(n_units * 32, dtype=torch.int32, device=cuda_device)
    unit_len = torch.empty(n_units, dtype=torch.int32, device=cuda_device)
    _lib.call("fvr_rplan_tile_rows", d.data_ptr(), n_views, w, h, tile[0], tile[1], 16, row_src.data_ptr(),
              unit_len.data_ptr(), _lib.stream_ptr())
    # restatement: tiles of tx x ty units; slots = the tile's rows in natural
    # order; slot k <- the tile's k-th longest row (ties in natural order)
    tx, ty = tile
    unit = np.arange(n_units)
    view, u = unit // (ux * uy), unit % (ux * uy)
    tiles_x, tiles_y = (ux + tx - 1) // tx, (uy + ty - 1) // ty
    tid = (view * tiles_y + (u // ux) // ty) * tiles_x + (u % ux) // tx
    tile_row = np.repeat(tid, 32)
    r = np.arange(n_units * 32)
    dest = np.lexsort((r, tile_row))
    src = np.lexsort((r, -row_len.astype(np.int64), tile_row))
    want = np.empty_like(r)
    want[dest] = src
    assert np.array_equal(row_src.cpu().numpy(), want)
    ul = row_len[want].reshape(n_units, 32).max(1)
    assert np.array_equal(unit_len.cpu().numpy(), (ul + 15) // 16 * 16)
