"""The library's host-side native passes, which run without a device:
fvr_copy_host_parallel (the parallel staging copy of frames) and
fvr_stage_inputs_host (inside voxels, bbox crops of images and masks, flame
counts per view: reconstruct.py:144-149, 299-301; volume.py:142-145), both
against numpy restatements."""

import ctypes

import numpy as np

from paper_1809_06417_b200 import _lib


def test_copy_host_parallel_concatenates():
    rng = np.random.default_rng(0)
    # sizes around the 1 MiB piece boundary, an empty buffer, odd lengths
    arrays = [rng.integers(0, 255, n, dtype=np.uint8) for n in (1 << 20, 3, 0, (1 << 21) + 7, 12_345)]
    total = sum(a.nbytes for a in arrays)
    dst = np.zeros(total, np.uint8)
    n = len(arrays)
    srcs = (ctypes.c_void_p * n)(*[a.ctypes.data for a in arrays])
    sizes = (ctypes.c_int64 * n)(*[a.nbytes for a in arrays])
    _lib.call("fvr_copy_host_parallel", ctypes.addressof(srcs), ctypes.addressof(sizes), n, dst.ctypes.data)
    assert np.array_equal(dst, np.concatenate(arrays))


def test_stage_inputs_host_matches_numpy():
    rng = np.random.default_rng(1)
    V, H, W = 3, 40, 50
    u0, v0, w, h = 7, 5, 31, 22
    full = (1 << V) - 1
    tags = rng.integers(0, full + 1, (9, 10, 11)).astype(np.uint32)
    images = [rng.random((H, W, 1), dtype=np.float32) * 255 for _ in range(V)]
    masks = [rng.random((H, W)) < 0.3 for _ in range(V)]
    n_vox = tags.size
    inside = np.zeros(n_vox, np.uint8)
    src = np.zeros((V, h, w), np.float32)
    mcrop = np.zeros((V, h, w), np.uint8)
    counts = np.zeros(V, np.int64)
    img_ptrs = (ctypes.c_void_p * V)(*[im.ctypes.data for im in images])
    img_rows = (ctypes.c_int64 * V)(*[im.strides[0] // 4 for im in images])
    bits = [np.ascontiguousarray(m) for m in masks]
    msk_ptrs = (ctypes.c_void_p * V)(*[b.ctypes.data for b in bits])
    msk_rows = (ctypes.c_int64 * V)(*[b.strides[0] for b in bits])
    _lib.call("fvr_stage_inputs_host", tags.ctypes.data, n_vox, full, V, ctypes.addressof(img_ptrs),
              ctypes.addressof(img_rows), images[0].strides[1] // 4, ctypes.addressof(msk_ptrs),
              ctypes.addressof(msk_rows), u0, v0, w, h, inside.ctypes.data, src.ctypes.data, mcrop.ctypes.data,
              counts.ctypes.data)
    assert np.array_equal(inside, (tags.ravel() == full).astype(np.uint8))
    for v in range(V):
        assert np.array_equal(src[v], images[v][v0:v0 + h, u0:u0 + w, 0])
        assert np.array_equal(mcrop[v], masks[v][v0:v0 + h, u0:u0 + w].astype(np.uint8))
        assert counts[v] == int(masks[v][v0:v0 + h, u0:u0 + w].sum())
