"""Shared pieces of the full-size parity checks (tests/test_gpu_fullsize.py and
tools/parity_curve.py): the device loop through the public API and the CPU
oracle loop on identical inputs, each recording the lattice every iteration
renders, so the error can be followed iteration by iteration."""

from __future__ import annotations

import os

import numpy as np

from tests.conftest import rel_err


def loop_cfg(sc, iters: int, deterministic: bool = True, seed: int = 0):
    from paper_1809_06417_b200 import ReconstructionConfig

    return ReconstructionConfig(alpha_l=0.006, alpha_d=1.0, tau=sc["tau"], max_iters=iters, converge_eps=1e-12,
                                deterministic_mode=deterministic, g_sigma=0.1, rng_seed=seed)


def device_loop(sc, iters: int, mode: str = "plan", record: bool = True, deterministic: bool = True, seed: int = 0):
    """reconstruct_channel on the device with FVR_RENDER=mode; returns
    (final lattice, rmse trace, [lattice rendered by iteration 1..iters])."""
    from paper_1809_06417_b200 import reconstruct_channel

    seen = []
    old = os.environ.get("FVR_RENDER")
    os.environ["FVR_RENDER"] = mode
    try:
        grid, trace = reconstruct_channel(
            sc["images"], sc["cams"], sc["geom"], sc["hull"], loop_cfg(sc, iters, deterministic, seed),
            render_cfg=sc["rcfg"], masks=sc["masks"], bbox=sc["bbox"],
            callback=(lambda it, g, r: seen.append(np.array(g.values, copy=True))) if record else None)
    finally:
        if old is None:
            os.environ.pop("FVR_RENDER", None)
        else:
            os.environ["FVR_RENDER"] = old
    return grid.values, np.array(trace.rmse), seen


def oracle_chunks(n: int) -> int:
    """Partial lattices of the oracle's adjust (16 in the reference); fewer
    when 16 f64 copies of the lattice would not fit comfortably in host RAM.
    The chunk count only changes the f64 summation order."""
    lattice = 8 * (n + 1) ** 3
    try:
        import psutil

        avail = psutil.virtual_memory().available
    except Exception:
        avail = 64 << 30
    for k in (16, 8, 4, 2):
        if k * lattice < avail // 4:
            return k
    return 1


def oracle_loop(sc, iters: int, record: bool = True):
    """oracle.cpu.reconstruct_channel (deterministic) on the same inputs."""
    from oracle import cpu
    from paper_1809_06417_b200.reconstruct import _init_grid

    b = sc["bbox"]
    cpu.set_threads(os.cpu_count() or 1)
    cpu.set_skip_empty(True)
    seen = []
    try:
        init = _init_grid(sc["geom"], sc["hull"], "green").values
        vals, rmse, _, secs = cpu.reconstruct_channel(
            [im.data[:, :, 0] for im in sc["images"]], sc["cams"], init, sc["hull"].inside_voxels(),
            [m.bits for m in sc["masks"]], (b.u0, b.v0, b.u1, b.v1), sc["geom"].origin, sc["geom"].edge,
            tau=sc["tau"], scattering=True, sigma_s=sc["rcfg"].sigma_s, scatter_dirs=sc["rcfg"].scatter_dirs,
            alpha_l=0.006, alpha_d_eff=loop_cfg(sc, iters).effective_alpha_d(sc["geom"]), max_iters=iters,
            converge_eps=1e-12, n_chunks=oracle_chunks(sc["n"]),
            callback=(lambda it, v, r: seen.append(np.array(v, copy=True))) if record else None)
    finally:
        cpu.set_skip_empty(False)
    return vals, np.array(rmse), seen, secs


def curve(dev, ref) -> dict:
    """Per-iteration parity of two recorded loops: max rel error of the
    lattice each iteration rendered, of the final lattice, and of the trace."""
    d_final, d_rmse, d_seen = dev
    r_final, r_rmse, r_seen = ref[:3]
    per_it = [rel_err(a, b) for a, b in zip(d_seen, r_seen)]
    return {"grid_rel_per_iter": per_it, "final_grid_rel": rel_err(d_final, r_final),
            "rmse_rel_per_iter": (np.abs(d_rmse - r_rmse) / np.abs(r_rmse)).tolist(),
            "rmse_dev": d_rmse.tolist(), "rmse_ref": r_rmse.tolist()}
