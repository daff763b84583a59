"""Operator layer with the signatures of fvr._kernels
(/root/reference/pkg/src/fvr/_kernels.py:25-306), backed by libfvr_b200.so.

Same arguments, same in-place outputs, same ``None`` return, numpy arrays in
host memory; each call stages through the device (``fvr_*_host`` entry
points).  ``adjust_rays_chunked`` deposits through the device's fixed-point
accumulator and adds the result into ``partials[0]`` -- the caller's
fixed-order merge over chunks therefore yields the same Δ up to the f32
deposit rounding (SURVEY.md §8c tolerance).  Thread-count knobs are accepted
for API compatibility: results never depend on them.
"""

from __future__ import annotations

import numpy as np

from . import _lib

MARCH_COUNT_EPS = 1e-9  # _kernels.py:25

_threads = 1


def set_threads(n: int) -> None:
    global _threads
    _threads = max(1, int(n))


def get_threads() -> int:
    return _threads


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _addr(a: np.ndarray) -> int:
    return a.ctypes.data


def _grid_from(shape_kp, grid_origin, edge) -> _lib.FvrGrid:
    g = _lib.FvrGrid()
    g.nx, g.ny, g.nz = (int(s) - 1 for s in shape_kp)
    for a in range(3):
        g.origin[a] = float(grid_origin[a])
    g.edge = float(edge)
    return g


def render_rays(origin, dirs, values, grid_origin, edge, tau, sigma_a, background, scattering,
                sigma_s, scat_dirs, phase_g, gather_dist, out):
    """Front-to-back under-blending of every ray; ``values`` (C, nx+1, ny+1,
    nz+1) f32, ``out`` (N, C) f64 written in place."""
    o = _f64(origin)
    d = _f64(dirs)
    v = np.ascontiguousarray(values, dtype=np.float32)
    bg = _f64(background)
    sd = _f64(scat_dirs)
    grid = _grid_from(v.shape[1:], grid_origin, edge)
    p = _lib.FvrRenderParams()
    p.tau, p.sigma_a, p.sigma_s, p.phase_g, p.gather_dist = tau, sigma_a, sigma_s, phase_g, gather_dist
    p.scattering = 1 if scattering else 0
    p.n_scat = int(sd.shape[0])
    res = np.empty((d.shape[0], v.shape[0]), dtype=np.float64)
    _lib.call("fvr_render_rays_host", _addr(o), _addr(d), d.shape[0], _addr(v), v.shape[0], grid, p,
              _addr(bg), _addr(sd), _addr(res))
    out[...] = res


def count_hull_samples(origin, dirs, inside_vox, grid_origin, edge, counts):
    """Per ray, the number of samples whose clamped cell is inside the hull."""
    o = _f64(origin)
    d = _f64(dirs)
    ins = np.ascontiguousarray(inside_vox, dtype=np.uint8)
    grid = _grid_from(tuple(s + 1 for s in ins.shape), grid_origin, edge)
    res = np.empty(d.shape[0], dtype=np.int64)
    _lib.call("fvr_count_hull_samples_host", _addr(o), _addr(d), d.shape[0], _addr(ins), grid, _addr(res))
    counts[...] = res


def adjust_rays_chunked(origin, dirs, residuals, g_values, g_offsets, use_g, inside_vox, grid_origin,
                        edge, tau, alpha_l, alpha_d, partials):
    """Back-project per-ray residuals onto the 8 key points of every in-hull
    sample (accumulated into ``partials`` in place)."""
    o = _f64(origin)
    d = _f64(dirs)
    r = _f64(residuals)
    gv = _f64(g_values)
    go = np.ascontiguousarray(g_offsets, dtype=np.int64)
    ins = np.ascontiguousarray(inside_vox, dtype=np.uint8)
    grid = _grid_from(partials.shape[1:], grid_origin, edge)
    if not (partials.flags.c_contiguous and partials.dtype == np.float64):
        raise ValueError("partials must be a C-contiguous float64 array")
    _lib.call("fvr_adjust_rays_host", _addr(o), _addr(d), d.shape[0], _addr(r), _addr(gv), _addr(go),
              1 if use_g else 0, _addr(ins), grid, float(tau), float(alpha_l), float(alpha_d),
              _addr(partials), int(partials.shape[0]))


__all__ = [
    "MARCH_COUNT_EPS",
    "set_threads",
    "get_threads",
    "render_rays",
    "count_hull_samples",
    "adjust_rays_chunked",
]
