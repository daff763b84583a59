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


def test_sell_layout_matches_restatement(cuda_device):
    """fvr_sell_layout = window order + per-slice padded max + exclusive scan
    + row_info + the count / ray-sample totals (engine._plan_count)."""
    import torch

    from paper_1809_06417_b200 import _lib

    rng = np.random.default_rng(7)
    for n, window, pad in ((100_003, 128, 8), (31, 32, 4), (4096, 1024, 8)):
        counts = rng.integers(0, 60, n).astype(np.int32)
        ray_samples = rng.integers(0, 9, 5001).astype(np.int32)
        d = torch.from_numpy(counts).to(cuda_device)
        rs = torch.from_numpy(ray_samples).to(cuda_device)
        ns = (n + 31) // 32
        row_of_pos = torch.empty(n, dtype=torch.int32, device=cuda_device)
        slice_len = torch.empty(ns, dtype=torch.int32, device=cuda_device)
        slice_off = torch.empty(ns + 1, dtype=torch.int64, device=cuda_device)
        row_info = torch.empty(n, dtype=torch.int64, device=cuda_device)
        totals = torch.empty(3, dtype=torch.int64, device=cuda_device)
        sid0 = torch.empty(rs.numel(), dtype=torch.int64, device=cuda_device)
        _lib.call("fvr_sell_layout", d.data_ptr(), n, window, pad, rs.data_ptr(), rs.numel(), sid0.data_ptr(),
                  row_of_pos.data_ptr(), slice_len.data_ptr(), slice_off.data_ptr(), row_info.data_ptr(),
                  totals.data_ptr(), _lib.stream_ptr())
        assert np.array_equal(sid0.cpu().numpy(), np.concatenate([[0], np.cumsum(ray_samples)[:-1]]))
        pos = np.arange(n)
        order = np.lexsort((pos, -counts.astype(np.int64), pos // window))
        assert np.array_equal(row_of_pos.cpu().numpy(), order)
        sl = np.zeros(ns * 32, np.int64)
        sl[:n] = counts[order]
        sl = sl.reshape(ns, 32).max(1)
        sl = (sl + pad - 1) // pad * pad
        assert np.array_equal(slice_len.cpu().numpy(), sl)
        off = np.concatenate([[0], np.cumsum(sl)])
        assert np.array_equal(slice_off.cpu().numpy(), off)
        rp = np.empty(n, np.int64)
        rp[order] = pos
        assert np.array_equal(row_info.cpu().numpy(), (off[rp >> 5] << 5) | (rp & 31))
        assert totals.cpu().tolist() == [int(off[-1]), int(counts.sum()), int(ray_samples.sum())]


@pytest.mark.parametrize("buckets", [24, 1, 5])
def test_rplan_layout_matches_restatement(cuda_device, buckets):
    """fvr_rplan_layout = tile rows + exclusive scan of the unit lengths +
    the unit order of fvr_rplan_unit_keys (engine._rplan_scan)."""
    import torch

    from paper_1809_06417_b200 import _lib

    rng = np.random.default_rng(buckets)
    n_views, w, h = 3, 139, 255
    ux, uy = (w + 7) // 8, (h + 3) // 4
    n_units = n_views * ux * uy
    row_len = rng.integers(0, 700, n_units * 32).astype(np.int32)
    d = torch.from_numpy(row_len).to(cuda_device)
    # restatement from the separately tested pieces
    rs_ref = torch.empty(n_units * 32, dtype=torch.int32, device=cuda_device)
    ul_ref = torch.empty(n_units, dtype=torch.int32, device=cuda_device)
    _lib.call("fvr_rplan_tile_rows", d.data_ptr(), n_views, w, h, 2, 4, 16, rs_ref.data_ptr(), ul_ref.data_ptr(),
              _lib.stream_ptr())
    ul = ul_ref.cpu().numpy().astype(np.int64)
    mx = torch.tensor([int(ul.max())], dtype=torch.int32, device=cuda_device)
    keys = torch.empty(n_units, dtype=torch.int64, device=cuda_device)
    _lib.call("fvr_rplan_unit_keys", ul_ref.data_ptr(), n_views, w, h, buckets, mx.data_ptr(), keys.data_ptr(),
              _lib.stream_ptr())
    order_ref = np.argsort(keys.cpu().numpy(), kind="stable")
    row_src = torch.empty(n_units * 32, dtype=torch.int32, device=cuda_device)
    unit_len = torch.empty(n_units, dtype=torch.int32, device=cuda_device)
    off = torch.empty(n_units + 1, dtype=torch.int64, device=cuda_device)
    order = torch.empty(n_units, dtype=torch.int32, device=cuda_device)
    totals = torch.empty(2, dtype=torch.int64, device=cuda_device)
    _lib.call("fvr_rplan_layout", d.data_ptr(), n_views, w, h, 2, 4, 16, buckets, row_src.data_ptr(),
              unit_len.data_ptr(), off.data_ptr(), order.data_ptr(), totals.data_ptr(), _lib.stream_ptr())
    assert np.array_equal(row_src.cpu().numpy(), rs_ref.cpu().numpy())
    assert np.array_equal(unit_len.cpu().numpy(), ul)
    assert np.array_equal(off.cpu().numpy(), np.concatenate([[0], np.cumsum(ul)]))
    assert np.array_equal(order.cpu().numpy(), order_ref)
    assert totals.cpu().tolist() == [int(ul.sum()), int(ul.max())]


def test_flame_rays_kp_map_morton_order(cuda_device):
    import torch

    from paper_1809_06417_b200 import _lib

    rng = np.random.default_rng(3)
    crops = (rng.random((5, 77, 131)) < 0.3).astype(np.uint8)
    d = torch.from_numpy(crops).to(cuda_device)
    n = int(crops.sum())
    rays = torch.empty(n, dtype=torch.int32, device=cuda_device)
    cnt = torch.empty(1, dtype=torch.int64, device=cuda_device)
    _lib.call("fvr_flame_rays", d.data_ptr(), 5, 131, 77, n, rays.data_ptr(), cnt.data_ptr(), _lib.stream_ptr())
    v, r, c = np.nonzero(crops)
    assert int(cnt.item()) == n
    assert np.array_equal(rays.cpu().numpy(), (v << 24) | (r * 131 + c))
    # count + select of nonzero bytes (the hull key-point list)
    flat = torch.from_numpy((rng.random(300_007) < 0.1).astype(np.uint8) * 7).to(cuda_device)
    c = torch.empty(1, dtype=torch.int64, device=cuda_device)
    _lib.call("fvr_count_nonzero_u8", flat.data_ptr(), flat.numel(), c.data_ptr(), _lib.stream_ptr())
    want_idx = np.flatnonzero(flat.cpu().numpy())
    assert int(c.item()) == want_idx.size
    sel = torch.empty(want_idx.size, dtype=torch.int32, device=cuda_device)
    _lib.call("fvr_select_nonzero_u8", flat.data_ptr(), flat.numel(), want_idx.size, sel.data_ptr(), c.data_ptr(),
              _lib.stream_ptr())
    assert np.array_equal(sel.cpu().numpy(), want_idx)
    # key-point map: position in the list, -1 elsewhere
    shape = (33, 40, 17)
    n_vox = int(np.prod(shape))
    kp = np.sort(rng.choice(n_vox, 5000, replace=False)).astype(np.int32)
    kp = kp[rng.permutation(kp.size)]
    dk = torch.from_numpy(kp).to(cuda_device)
    m = torch.empty(n_vox, dtype=torch.int32, device=cuda_device)
    _lib.call("fvr_kp_map", dk.data_ptr(), kp.size, n_vox, m.data_ptr(), _lib.stream_ptr())
    want = np.full(n_vox, -1, np.int32)
    want[kp] = np.arange(kp.size)
    assert np.array_equal(m.cpu().numpy(), want)
    # Morton order of the permuted list
    out = torch.empty_like(dk)
    g = _lib.FvrGrid()
    g.nx, g.ny, g.nz = shape[0] - 1, shape[1] - 1, shape[2] - 1
    g.edge = 1.0
    _lib.call("fvr_morton_order", dk.data_ptr(), kp.size, g, out.data_ptr(), _lib.stream_ptr())
    mk = _morton_ref(kp.astype(np.int64), shape)
    assert np.array_equal(out.cpu().numpy(), kp[np.argsort(mk, kind="stable")])


def _dist_ref(values, force, cap=30):
    """fvr_occupancy restated: seed 0 at positive or forced key points (cap + 1
    elsewhere), then the separable z, y, x passes min_d max(|d|, f) over
    |d| <= cap inside the lattice."""
    m = (values > 0).any(0) | force.astype(bool)
    f = np.where(m, 0, cap + 1).astype(np.int64)
    for axis in (2, 1, 0):
        out = f.copy()
        n = f.shape[axis]
        for dd in range(1, cap + 1):
            if dd >= n:
                break
            lo = [slice(None)] * 3
            hi = [slice(None)] * 3
            lo[axis], hi[axis] = slice(dd, None), slice(None, n - dd)
            # neighbour at p - dd for positions p >= dd, and at p + dd for p < n - dd
            out[tuple(lo)] = np.minimum(out[tuple(lo)], np.maximum(dd, f[tuple(hi)]))
            out[tuple(hi)] = np.minimum(out[tuple(hi)], np.maximum(dd, f[tuple(lo)]))
        f = out
    return f.astype(np.uint8)


@pytest.mark.parametrize("shape", [(33, 70, 17), (65, 65, 65), (129, 40, 129)])
def test_occupancy_distance_map(cuda_device, shape):
    import torch

    from paper_1809_06417_b200 import _lib

    rng = np.random.default_rng(shape[1])
    values = np.where(rng.random((2,) + shape) < 0.002, 1.0, -1.0).astype(np.float32)
    force = (rng.random(shape) < 0.001).astype(np.uint8)
    g = _lib.FvrGrid()
    g.nx, g.ny, g.nz = shape[0] - 1, shape[1] - 1, shape[2] - 1
    g.edge = 1.0
    dv = torch.from_numpy(values).to(cuda_device)
    df = torch.from_numpy(force).to(cuda_device)
    occ = torch.empty(shape, dtype=torch.uint8, device=cuda_device)
    _lib.call("fvr_occupancy", dv.data_ptr(), 2, df.data_ptr(), g, occ.data_ptr(), _lib.stream_ptr())
    assert np.array_equal(occ.cpu().numpy(), _dist_ref(values, force))


def test_plan_row_sort(cuda_device):
    """fvr_plan_sort_rows: every lane-row of a 6-byte SELL slice sorted by its
    24-bit column, the weight (exponent byte + mantissa half) travelling with
    it; slices longer than 1024 entries are left alone."""
    import torch

    from paper_1809_06417_b200 import _lib

    rng = np.random.default_rng(7)
    lens = np.array([8, 40, 1032, 16], dtype=np.int32)  # multiples of 8; the third is too long to sort
    offs = np.concatenate([[0], np.cumsum(lens.astype(np.int64))])
    total = int(offs[-1])
    # per (slice, lane, position): column, exponent, half
    col = rng.integers(0, 1 << 24, size=(32 * total,), dtype=np.uint32)
    ex = rng.integers(100, 140, size=(32 * total,), dtype=np.uint32)
    half = rng.integers(0, 1 << 16, size=(32 * total,), dtype=np.uint32)
    a = np.zeros(32 * total, dtype=np.uint32)
    b = np.zeros(32 * total, dtype=np.uint16)
    where = {}
    for s, (ln_, off) in enumerate(zip(lens, offs[:-1])):
        for lane in range(32):
            for p in range(ln_):
                ia = (((off >> 2) + (p >> 2)) * 32 + lane) * 4 + (p & 3)
                ib = (((off >> 3) + (p >> 3)) * 32 + lane) * 8 + (p & 7)
                where[(s, lane, p)] = (ia, ib)
    keys = np.arange(32 * total)
    for (s, lane, p), (ia, ib) in where.items():
        a[ia] = col[keys[ia]] | (ex[keys[ia]] << 24)
        b[ib] = half[keys[ia]]
    dev = torch.device("cuda", 0)
    ta = torch.from_numpy(a.view(np.int32).copy()).to(dev)
    tb = torch.from_numpy(np.ascontiguousarray(b).view(np.int32).copy()).to(dev)
    sl = torch.from_numpy(lens).to(dev)
    so = torch.from_numpy(offs[:-1].copy()).to(dev)
    _lib.call("fvr_plan_sort_rows", sl.data_ptr(), so.data_ptr(), len(lens), ta.data_ptr(), tb.data_ptr(),
              _lib.stream_ptr())
    ga = ta.cpu().numpy().view(np.uint32)
    gb = tb.cpu().numpy().view(np.uint16)
    for s, (ln_, off) in enumerate(zip(lens, offs[:-1])):
        for lane in range(32):
            idx = [where[(s, lane, p)] for p in range(ln_)]
            before = sorted((int(a[ia]) & 0xFFFFFF, int(a[ia]) >> 24, int(b[ib])) for ia, ib in idx)
            after = [(int(ga[ia]) & 0xFFFFFF, int(ga[ia]) >> 24, int(gb[ib])) for ia, ib in idx]
            if ln_ > 1024:
                assert [(int(a[ia]), int(b[ib])) for ia, ib in idx] == [(int(ga[ia]), int(gb[ib])) for ia, ib in idx]
            else:
                assert after == before


def test_sell_pad_zero(cuda_device):
    """fvr_sell_pad_zero clears exactly the padding of each lane-row (from the
    fill's cursor to the slice length) and leaves the filled entries alone."""
    import torch

    from paper_1809_06417_b200 import _lib

    rng = np.random.default_rng(11)
    lens = np.array([8, 16, 24], dtype=np.int32)
    offs = np.concatenate([[0], np.cumsum(lens.astype(np.int64))])
    total = int(offs[-1])
    n_rows = 3 * 32 - 5  # the last slice is partly unused
    row_of_pos = rng.permutation(n_rows).astype(np.int32)
    cursor = np.zeros(n_rows, dtype=np.int64)
    for pos in range(n_rows):
        cursor[row_of_pos[pos]] = rng.integers(0, lens[pos >> 5] + 1)
    a = np.full(32 * total, 0xDEADBEEF, dtype=np.uint32)
    b = np.full(32 * total, 0xBEEF, dtype=np.uint16)
    dev = torch.device("cuda", 0)
    ta = torch.from_numpy(a.view(np.int32).copy()).to(dev)
    tb = torch.from_numpy(b.view(np.int32).copy()).to(dev)
    args = [torch.from_numpy(x).to(dev) for x in (cursor, row_of_pos, lens, offs[:-1].copy())]
    _lib.call("fvr_sell_pad_zero", args[0].data_ptr(), args[1].data_ptr(), n_rows, args[2].data_ptr(),
              args[3].data_ptr(), len(lens), ta.data_ptr(), tb.data_ptr(), _lib.stream_ptr())
    ga = ta.cpu().numpy().view(np.uint32)
    gb = tb.cpu().numpy().view(np.uint16)
    for pos in range(3 * 32):
        s, lane = pos >> 5, pos & 31
        off, ln_ = int(offs[s]), int(lens[s])
        c = int(cursor[row_of_pos[pos]]) if pos < n_rows else 0
        for p in range(ln_):
            ia = (((off >> 2) + (p >> 2)) * 32 + lane) * 4 + (p & 3)
            ib = (((off >> 3) + (p >> 3)) * 32 + lane) * 8 + (p & 7)
            if p < c:
                assert ga[ia] == 0xDEADBEEF and gb[ib] == 0xBEEF
            else:
                assert ga[ia] == 0 and gb[ib] == 0
