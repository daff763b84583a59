"""CPU oracle for the B200 path -- TEST INFRASTRUCTURE ONLY.

Restates the reference's algorithm (/root/reference/pkg/src/fvr/) on the CPU:
the three kernels in C (fvr_oracle.c, OpenMP, IEEE fp64 without FMA
contraction, bit-identical to the numba build) and the host glue in numpy
with the reference's own expressions.  Only tests/, __graft_entry__.smoke()
and bench.py (the ``cpu_baseline`` leg and ``--impl reference``) may import
this module; the product package never does.

Parity pinning: tests/test_oracle_golden.py checks every function here
against golden vectors produced by running the reference itself
(tests/golden/make_golden.py, committed with its outputs).

Functions and the reference lines they follow:
  pixel_rays             geometry.py:125-137
  fibonacci_sphere       radiometry.py:222-230
  render_rays            _kernels.py:101-186   (C)
  count_hull_samples     _kernels.py:189-224   (C)
  adjust_rays_chunked    _kernels.py:227-306   (C)
  render_pixels          render.py:183-217
  adjust_pass            reconstruct.py:152-227
  reconstruct_channel    reconstruct.py:250-334 (deterministic or numpy-drawn G)
  key_point_mask         volume.py:146-164
  visual_hull            volume.py:249-328
  color_temp_table       radiometry.py:48-64, 173-203
  temp_from_green        radiometry.py:206-219
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
MARCH_COUNT_EPS = 1e-9

_lib = None


def build(force: bool = False) -> str:
    """Compile fvr_oracle.c (gcc -O2 -fopenmp -ffp-contract=off)."""
    src = os.path.join(HERE, "fvr_oracle.c")
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", HERE])
    return LIB


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB)
        P, I64, D, I = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_int
        L.oracle_render_rays.argtypes = [P, P, I64, P, I, I, I, I, P, D, D, D, P, I, D, P, I, D, D, P]
        L.oracle_render_rays.restype = None
        L.oracle_count_hull_samples.argtypes = [P, P, I64, P, I, I, I, P, D, P]
        L.oracle_count_hull_samples.restype = None
        L.oracle_adjust_rays_chunked.argtypes = [P, P, I64, P, P, P, I, P, I, I, I, P, D, D, D, D, P, I]
        L.oracle_adjust_rays_chunked.restype = None
        L.oracle_set_threads.argtypes = [I]
        L.oracle_set_threads.restype = I
        L.oracle_get_threads.restype = I
        L.oracle_set_skip_empty.argtypes = [I]
        L.oracle_set_skip_empty.restype = I
        _lib = L
    return _lib


def set_threads(n: int) -> int:
    return lib().oracle_set_threads(int(n))


def get_threads() -> int:
    return lib().oracle_get_threads()


def set_skip_empty(on: bool) -> bool:
    """Exact empty-space skip in render_rays (fvr_oracle.c): samples whose
    reads touch only non-positive key points add exactly zero, so skipping
    them is bit-identical (tests/test_oracle_golden.py checks it).  Off by
    default; the full-size parity tests turn it on to fit their time budget."""
    return bool(lib().oracle_set_skip_empty(int(bool(on))))


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def _p(a: np.ndarray) -> int:
    return a.ctypes.data


# --- kernels (C) -----------------------------------------------------------------


def render_rays(origin, dirs, values, grid_origin, edge, tau, sigma_a, background, scattering,
                sigma_s, scat_dirs, phase_g, gather_dist) -> np.ndarray:
    o, d = _c(origin, np.float64), _c(dirs, np.float64)
    v = _c(values, np.float32)
    go, bg, sd = _c(grid_origin, np.float64), _c(background, np.float64), _c(scat_dirs, np.float64)
    nch, nx1, ny1, nz1 = v.shape
    out = np.empty((d.shape[0], nch))
    lib().oracle_render_rays(_p(o), _p(d), d.shape[0], _p(v), nch, nx1 - 1, ny1 - 1, nz1 - 1, _p(go),
                             float(edge), float(tau), float(sigma_a), _p(bg), int(bool(scattering)),
                             float(sigma_s), _p(sd), sd.shape[0], float(phase_g), float(gather_dist),
                             _p(out))
    return out


def count_hull_samples(origin, dirs, inside_vox, grid_origin, edge) -> np.ndarray:
    o, d = _c(origin, np.float64), _c(dirs, np.float64)
    ins = _c(inside_vox, np.uint8)
    go = _c(grid_origin, np.float64)
    counts = np.empty(d.shape[0], dtype=np.int64)
    lib().oracle_count_hull_samples(_p(o), _p(d), d.shape[0], _p(ins), *ins.shape, _p(go), float(edge),
                                    _p(counts))
    return counts


def adjust_rays_chunked(origin, dirs, residuals, g_values, g_offsets, use_g, inside_vox, grid_origin,
                        edge, tau, alpha_l, alpha_d, partials) -> None:
    o, d = _c(origin, np.float64), _c(dirs, np.float64)
    r, gv = _c(residuals, np.float64), _c(g_values, np.float64)
    goff = _c(g_offsets, np.int64)
    ins = _c(inside_vox, np.uint8)
    go = _c(grid_origin, np.float64)
    assert partials.flags.c_contiguous and partials.dtype == np.float64
    lib().oracle_adjust_rays_chunked(_p(o), _p(d), d.shape[0], _p(r), _p(gv), _p(goff), int(bool(use_g)),
                                     _p(ins), *ins.shape, _p(go), float(edge), float(tau), float(alpha_l),
                                     float(alpha_d), _p(partials), partials.shape[0])


# --- host glue (numpy) ------------------------------------------------------------


def camera_center(cam) -> np.ndarray:
    return -cam.rotation.T @ cam.translation


def pixel_rays(cam, us, vs):
    us = np.asarray(us, dtype=np.float64).ravel()
    vs = np.asarray(vs, dtype=np.float64).ravel()
    d = np.stack([(us - cam.cx) / cam.fx, (vs - cam.cy) / cam.fy, np.ones_like(us)], axis=1)
    d = d @ cam.rotation
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    return camera_center(cam), d


def fibonacci_sphere(n: int) -> np.ndarray:
    i = np.arange(n, dtype=np.float64)
    z = 1.0 - (2.0 * i + 1.0) / n
    phi = i * np.pi * (3.0 - np.sqrt(5.0))
    r = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    return np.stack([r * np.cos(phi), r * np.sin(phi), z], axis=1)


def render_pixels(cam, planes, grid_origin, edge, tau, sigma_a, background, us, vs, scattering=False,
                  sigma_s=0.0, scatter_dirs=32, phase_g=0.0) -> np.ndarray:
    """planes: (C, nx+1, ny+1, nz+1); background: (C,) -> (N, C) f64."""
    origin, dirs = pixel_rays(cam, us, vs)
    scat = fibonacci_sphere(scatter_dirs) if scattering else np.zeros((1, 3))
    return render_rays(origin, dirs, planes, grid_origin, edge, tau, sigma_a, background, scattering,
                       sigma_s, scat, phase_g, edge)


def render_view(cam, planes, grid_origin, edge, tau, sigma_a, background, **kw) -> np.ndarray:
    uu, vv = np.meshgrid(np.arange(cam.width, dtype=np.float64) + 0.5,
                         np.arange(cam.height, dtype=np.float64) + 0.5, indexing="xy")
    out = render_pixels(cam, planes, grid_origin, edge, tau, sigma_a, background, uu.ravel(), vv.ravel(), **kw)
    return out.reshape(cam.height, cam.width, -1).astype(np.float32)


def key_point_mask(inside: np.ndarray) -> np.ndarray:
    nx, ny, nz = inside.shape
    kp = np.zeros((nx + 1, ny + 1, nz + 1), dtype=bool)
    for dx in (0, 1):
        for dy in (0, 1):
            for dz in (0, 1):
                kp[dx:dx + nx, dy:dy + ny, dz:dz + nz] |= inside
    return kp


def adjust_pass(values, inside, cams, residuals, masks, bbox, grid_origin, edge, tau, alpha_l,
                alpha_d_eff, n_chunks=16, rng=None, g_sigma=0.1) -> np.ndarray:
    """adjust_pass (reconstruct.py:152-227); bbox = (u0, v0, u1, v1).  With
    ``rng`` (a numpy Generator) the stochastic G = clip(N(1, g_sigma), 0, 2)
    is drawn view-major, row-major, front to back (reconstruct.py:191-204);
    without it, deterministic mode.  Returns new values."""
    u0, v0, u1, v1 = bbox
    ins = np.ascontiguousarray(inside, dtype=np.uint8)
    partials = np.zeros((n_chunks,) + values.shape)
    for cam, res, mask in zip(cams, residuals, masks):
        window = np.zeros_like(mask)
        window[v0:v1 + 1, u0:u1 + 1] = True
        rows, cols = np.nonzero(mask & window)
        if rows.size == 0:
            continue
        origin, dirs = pixel_rays(cam, cols + 0.5, rows + 0.5)
        offsets = np.zeros(rows.size, np.int64)
        g_values, use_g = np.ones(1), False
        if rng is not None and g_sigma != 0.0:
            counts = count_hull_samples(origin, dirs, ins, grid_origin, edge)
            np.cumsum(counts[:-1], out=offsets[1:])
            total = int(offsets[-1] + counts[-1])
            g_values = np.clip(rng.normal(1.0, g_sigma, size=total), 0.0, 2.0) if total else np.ones(1)
            use_g = True
        adjust_rays_chunked(origin, dirs, np.asarray(res, np.float64)[rows, cols], g_values, offsets, use_g,
                            ins, grid_origin, edge, tau, alpha_l, alpha_d_eff, partials)
    delta = np.zeros(values.shape)
    for c in range(n_chunks):
        delta += partials[c]
    new = values.astype(np.float64) + delta
    np.maximum(new, -1.0, out=new)
    return new.astype(np.float32)


def reconstruct_channel(src_images, cams, values, inside, masks, bbox, grid_origin, edge, *, tau,
                        sigma_a=1.0, background=0.0, scattering=False, sigma_s=0.0, scatter_dirs=32,
                        alpha_l, alpha_d_eff, max_iters, converge_eps, n_chunks=16, callback=None,
                        stochastic_seed=None, g_sigma=0.1):
    """reconstruct.py:250-334 in deterministic mode. src_images: list of (H, W)
    f32; values: initial lattice f32. Returns (values, rmse list, converged, s/it).
    ``callback(it, values, rmse)`` sees each iteration's rendered lattice
    (before its adjust), as the reference's callback does (reconstruct.py:316).
    ``stochastic_seed``: the reference's default mode, G drawn from
    np.random.default_rng(seed) (reconstruct.py:296)."""
    rng = None if stochastic_seed is None else np.random.default_rng(stochastic_seed)
    u0, v0, u1, v1 = bbox
    us = np.arange(u0, u1 + 1, dtype=np.float64) + 0.5
    vs = np.arange(v0, v1 + 1, dtype=np.float64) + 0.5
    uu, vv = np.meshgrid(us, vs, indexing="xy")
    uu, vv = uu.ravel(), vv.ravel()
    h_bb, w_bb = v1 - v0 + 1, u1 - u0 + 1
    src_blocks = [np.asarray(im)[v0:v1 + 1, u0:u1 + 1].astype(np.float64) for im in src_images]
    values = np.ascontiguousarray(values, dtype=np.float32).copy()
    rmses, prev, converged = [], None, False
    t0 = time.perf_counter()
    for _ in range(max_iters):
        recs, per_view = [], []
        for cam, src in zip(cams, src_blocks):
            rec = render_pixels(cam, values[None], grid_origin, edge, tau, sigma_a, np.array([background]),
                                uu, vv, scattering=scattering, sigma_s=sigma_s,
                                scatter_dirs=scatter_dirs).reshape(h_bb, w_bb)
            recs.append(rec)
            per_view.append(float(np.sqrt(np.mean((src - rec) ** 2))))
        rmse = float(np.mean(per_view))
        rmses.append(rmse)
        if callback is not None:
            callback(len(rmses), values, rmse)
        if rmse < converge_eps or (prev is not None and abs(rmse - prev) < converge_eps):
            converged = True
            break
        prev = rmse
        residuals = []
        for src, rec, cam in zip(src_blocks, recs, cams):
            f = np.zeros((cam.height, cam.width))
            f[v0:v1 + 1, u0:u1 + 1] = src - rec
            residuals.append(f)
        values = adjust_pass(values, inside, cams, residuals, masks, bbox, grid_origin, edge, tau, alpha_l,
                             alpha_d_eff, n_chunks, rng=rng, g_sigma=g_sigma)
    secs = (time.perf_counter() - t0) / max(len(rmses), 1)
    return values, rmses, converged, secs


def visual_hull(nx, ny, nz, grid_origin, edge, masks, cams) -> np.ndarray:
    """Hull tags (nx, ny, nz) u32 (volume.py:249-328)."""
    counts = (nx, ny, nz)
    xs = grid_origin[0] + edge * np.arange(nx + 1)
    ys = grid_origin[1] + edge * np.arange(ny + 1)
    zs = grid_origin[2] + edge * np.arange(nz + 1)
    kp = np.stack(np.meshgrid(xs, ys, zs, indexing="ij"), axis=-1).reshape(-1, 3)
    lat = (nx + 1, ny + 1, nz + 1)
    tags = np.zeros(counts, dtype=np.uint32)
    for i, (mask, cam) in enumerate(zip(masks, cams)):
        mask = np.asarray(mask, dtype=bool)
        pts = kp @ cam.rotation.T + cam.translation
        z = pts[:, 2]
        ok = z > 0
        zs_ = np.where(ok, z, 1.0)
        u = (cam.fx * pts[:, 0] / zs_ + cam.cx).reshape(lat)
        v = (cam.fy * pts[:, 1] / zs_ + cam.cy).reshape(lat)
        ok = ok.reshape(lat)
        umin = np.full(counts, np.inf)
        umax = np.full(counts, -np.inf)
        vmin = np.full(counts, np.inf)
        vmax = np.full(counts, -np.inf)
        vox_ok = np.ones(counts, dtype=bool)
        for dx in (0, 1):
            for dy in (0, 1):
                for dz in (0, 1):
                    sl = (slice(dx, dx + nx), slice(dy, dy + ny), slice(dz, dz + nz))
                    umin = np.minimum(umin, u[sl])
                    umax = np.maximum(umax, u[sl])
                    vmin = np.minimum(vmin, v[sl])
                    vmax = np.maximum(vmax, v[sl])
                    vox_ok &= ok[sl]
        W, H = cam.width, cam.height
        iu0 = np.clip(np.floor(umin).astype(np.int64), 0, W - 1)
        iu1 = np.clip(np.ceil(umax).astype(np.int64) - 1, 0, W - 1)
        iv0 = np.clip(np.floor(vmin).astype(np.int64), 0, H - 1)
        iv1 = np.clip(np.ceil(vmax).astype(np.int64) - 1, 0, H - 1)
        off = (umax <= 0) | (umin >= W) | (vmax <= 0) | (vmin >= H)
        sat = np.zeros((H + 1, W + 1), dtype=np.int64)
        sat[1:, 1:] = np.cumsum(np.cumsum(mask, axis=0), axis=1)
        hit = (sat[iv1 + 1, iu1 + 1] - sat[iv0, iu1 + 1] - sat[iv1 + 1, iu0] + sat[iv0, iu0]) > 0
        tags[hit & vox_ok & ~off] |= np.uint32(1 << i)
    return tags


# CIE 1931 2-degree observer (x̄, ȳ, z̄ at 380..780 nm, 5 nm); same table as
# paper_1809_06417_b200/csrc/fvr_temp.cu, checked against the reference's
# cie_data.py by tests/test_oracle_golden.py.
def _cie_table() -> np.ndarray:
    import re

    src = open(os.path.join(HERE, "..", "paper_1809_06417_b200", "csrc", "fvr_temp.cu")).read()
    cols = []
    for name in ("kCieX", "kCieY", "kCieZ"):
        body = re.search(name + r"\[81\] = \{(.*?)\};", src, re.S).group(1)
        cols.append([float(x) for x in body.replace("\n", " ").split(",")])
    lam = 380.0 + 5.0 * np.arange(81)
    return np.column_stack([lam] + cols)


XYZ_TO_SRGB = np.array([[3.2404542, -1.5371385, -0.4985314],
                        [-0.9692660, 1.8760108, 0.0415560],
                        [0.0556434, -0.2040259, 1.0572252]])


def color_temp_table(t_min=1000.0, t_max=2300.0, step=1.0):
    """(temperatures, entries (N, 3)) of the black-body map."""
    h, c, k = 6.62607015e-34, 299792458.0, 1.380649e-23
    n = int(np.floor((t_max - t_min) / step + 1e-9))
    temps = t_min + step * np.arange(n + 1)
    if temps[-1] < t_max - 1e-9 * t_max:
        temps = np.append(temps, t_max)
    cie = _cie_table()
    lam = cie[:, 0] * 1e-9
    lam2 = lam[None, :]
    T = temps[:, None]
    x = h * c / (lam2 * k * T)
    amp = 2.0 * h * c**2 / lam2**5
    with np.errstate(over="ignore", under="ignore"):
        L = np.where(x > 700.0, amp * np.exp(-np.minimum(x, 1e6)), amp / np.expm1(x))
    xyz = np.stack([np.trapezoid(L * cie[:, 1 + j][None, :], lam, axis=1) for j in range(3)], axis=1)
    rgb = np.maximum(xyz @ XYZ_TO_SRGB.T, 0.0)
    return temps, rgb / rgb.max() * 255.0


def temp_from_green(green, temps, g):
    g = np.asarray(g, dtype=np.float64)
    clamped = (g < green[0]) | (g > green[-1])
    return np.interp(np.clip(g, green[0], green[-1]), green, temps), clamped


def bracket_index(green, g) -> np.ndarray:
    """np.interp's bracket: largest j with green[j] <= clip(g)."""
    gc = np.clip(np.asarray(g, dtype=np.float64), green[0], green[-1])
    return np.clip(np.searchsorted(green, gc, side="right") - 1, 0, green.size - 1).astype(np.int32)
