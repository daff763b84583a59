"""Pin the CPU oracle against golden vectors produced by the reference itself
(tests/golden/make_golden.py).  Integer outputs must be equal; fp64 outputs
are expected bit-identical (same expression order, no FMA) and are checked
with a 1e-12 relative guard that reports the exact-match fraction."""

import numpy as np
import pytest

from oracle import cpu
from paper_1809_06417_b200.geometry import Camera
from paper_1809_06417_b200.volume import HullTags
from tests.conftest import cameras_from, load_golden, rel_err


@pytest.fixture(scope="module")
def kern():
    return load_golden("kernels.npz")


@pytest.mark.parametrize("name,scat,sig,g,nd", [("plain", False, 0.0, 0.0, 1),
                                                ("scat", True, 0.3, 0.0, 32),
                                                ("scat_g", True, 0.3, 0.4, 16)])
def test_render_rays_matches_reference(kern, name, scat, sig, g, nd):
    sd = cpu.fibonacci_sphere(nd) if scat else np.zeros((1, 3))
    out = cpu.render_rays(kern["origin"], kern["dirs"], kern["values"], kern["lo"], float(kern["edge"]), 0.05, 1.0,
                          kern["background"], scat, sig, sd, g, float(kern["edge"]))
    ref = kern["render_" + name]
    assert np.array_equal(out, ref), f"exact {np.mean(out == ref):.4f}, rel {rel_err(out, ref):.3e}"


def test_render_rays_origin_inside_box(kern):
    out = cpu.render_rays(kern["inner"], kern["dirs"], kern["values"], kern["lo"], float(kern["edge"]), 0.05, 1.0,
                          kern["background"], False, 0.0, np.zeros((1, 3)), 0.0, float(kern["edge"]))
    assert np.array_equal(out, kern["render_inner"])


def test_count_hull_samples_matches_reference(kern):
    counts = cpu.count_hull_samples(kern["origin"], kern["dirs"], kern["inside"], kern["lo"], float(kern["edge"]))
    assert np.array_equal(counts, kern["counts"])


@pytest.mark.parametrize("use_g", [False, True])
def test_adjust_matches_reference(kern, use_g):
    n = int(kern["n"])
    parts = np.zeros((16, n + 1, n + 1, n + 1))
    gv = kern["g_values"] if use_g else np.ones(1)
    go = kern["g_offsets"] if use_g else np.zeros(kern["dirs"].shape[0], np.int64)
    cpu.adjust_rays_chunked(kern["origin"], kern["dirs"], kern["residuals"], gv, go, use_g, kern["inside"],
                            kern["lo"], float(kern["edge"]), 0.05, 0.006, 1.0, parts)
    ref = kern["adjust_g" if use_g else "adjust_det"]
    got = parts.sum(axis=0)
    assert np.array_equal(got, ref), f"rel {rel_err(got, ref):.3e}"


def test_thread_count_does_not_change_results(kern):
    before = cpu.get_threads()
    outs = []
    try:
        for n in (1, 3, 8):
            cpu.set_threads(n)
            outs.append(cpu.render_rays(kern["origin"], kern["dirs"], kern["values"], kern["lo"],
                                        float(kern["edge"]), 0.05, 1.0, kern["background"], False, 0.0,
                                        np.zeros((1, 3)), 0.0, float(kern["edge"])))
    finally:
        cpu.set_threads(before)
    assert all(np.array_equal(outs[0], o) for o in outs[1:])


def test_render_view_matches_reference():
    g = load_golden("render.npz")
    cam = cameras_from(g, Camera)[0]
    plain = cpu.render_view(cam, g["values"], g["origin"], float(g["edge"]), 0.05, 1.0, np.array([1.0, 2.0, 3.0]))
    assert np.array_equal(plain, g["plain"])
    scat = cpu.render_view(cam, g["values"], g["origin"], float(g["edge"]), 0.05, 1.0, np.zeros(3),
                           scattering=True, sigma_s=0.3, scatter_dirs=32)
    assert np.array_equal(scat, g["scat"])


@pytest.mark.parametrize("fixture", ["config1.npz", "loop_scatter.npz"])
def test_hull_matches_reference(fixture):
    g = load_golden(fixture)
    cams = cameras_from(g, Camera)
    n = int(g["n"])
    tags = cpu.visual_hull(n, n, n, g["origin"], float(g["edge"]), list(g["masks"]), cams)
    assert np.array_equal(tags, g["hull_tags"])


@pytest.mark.parametrize("fixture", ["config1.npz", "loop_scatter.npz"])
def test_reconstruct_channel_matches_reference(fixture):
    g = load_golden(fixture)
    cams = cameras_from(g, Camera)
    hull = HullTags(g["hull_tags"], len(cams))
    kp = hull.key_point_mask()
    init = np.where(kp, np.float32(0.0), np.float32(-1.0))
    vals, rmse, conv, _ = cpu.reconstruct_channel(
        [im[:, :, 1] for im in g["blanked"]], cams, init, hull.inside_voxels(), list(g["masks"]), tuple(g["bbox"]),
        g["origin"], float(g["edge"]), tau=float(g["tau"]), scattering=bool(g["scattering"]),
        sigma_s=float(g["sigma_s"]), alpha_l=0.006, alpha_d_eff=float(g["alpha_d_eff"]),
        max_iters=int(g["iters"]), converge_eps=1e-12)
    assert conv == bool(g["converged"])
    assert np.array_equal(np.array(rmse), g["rmse"]), np.max(np.abs(np.array(rmse) - g["rmse"]))
    assert np.array_equal(vals, g["green"]), f"exact {np.mean(vals == g['green']):.5f} rel {rel_err(vals, g['green']):.2e}"


def test_color_temp_table_matches_reference():
    g = load_golden("ctmap.npz")
    assert np.array_equal(cpu._cie_table(), g["cie"])
    temps, entries = cpu.color_temp_table(1000.0, 2300.0, 1.0)
    assert np.array_equal(temps, g["temps"])
    assert np.array_equal(entries, g["entries"])
    t2, e2 = cpu.color_temp_table(1000.0, 1999.5, 3.0)
    assert np.array_equal(t2, g["odd_temps"])
    assert np.array_equal(e2, g["odd_entries"])


def test_temp_from_green_matches_reference():
    g = load_golden("ctmap.npz")
    T, clamped = cpu.temp_from_green(g["entries"][:, 1], g["temps"], g["greens"])
    assert np.array_equal(T, g["T"])
    assert np.array_equal(clamped, g["clamped"])


@pytest.mark.parametrize("fixture", ["config1.npz", "loop_scatter.npz"])
def test_empty_space_skip_is_bit_identical(fixture):
    """The opt-in exact skip (used by the full-size parity tests) leaves every
    bit of the reference's loop unchanged, with and without scattering."""
    g = load_golden(fixture)
    cams = cameras_from(g, Camera)
    hull = HullTags(g["hull_tags"], len(cams))
    init = np.where(hull.key_point_mask(), np.float32(0.0), np.float32(-1.0))
    cpu.set_skip_empty(True)
    try:
        vals, rmse, _, _ = cpu.reconstruct_channel(
            [im[:, :, 1] for im in g["blanked"]], cams, init, hull.inside_voxels(), list(g["masks"]),
            tuple(g["bbox"]), g["origin"], float(g["edge"]), tau=float(g["tau"]), scattering=bool(g["scattering"]),
            sigma_s=float(g["sigma_s"]), alpha_l=0.006, alpha_d_eff=float(g["alpha_d_eff"]),
            max_iters=int(g["iters"]), converge_eps=1e-12)
        scat = cpu.render_view(cams[0], g["truth"], g["origin"], float(g["edge"]), float(g["tau"]), 1.0,
                               np.zeros(3), scattering=True, sigma_s=0.3, scatter_dirs=32)
    finally:
        cpu.set_skip_empty(False)
    assert np.array_equal(np.array(rmse), g["rmse"])
    assert np.array_equal(vals, g["green"])
    ref = cpu.render_view(cams[0], g["truth"], g["origin"], float(g["edge"]), float(g["tau"]), 1.0, np.zeros(3),
                          scattering=True, sigma_s=0.3, scatter_dirs=32)
    assert np.array_equal(scat, ref)


def test_stochastic_loop_matches_reference():
    """The reference's default mode: G drawn from default_rng(seed) per
    in-hull sample, view-major, front to back (reconstruct.py:191-204)."""
    g = load_golden("config1.npz")
    s = load_golden("stochastic.npz")
    cams = cameras_from(g, Camera)
    hull = HullTags(g["hull_tags"], len(cams))
    init = np.where(hull.key_point_mask(), np.float32(0.0), np.float32(-1.0))
    vals, rmse, _, _ = cpu.reconstruct_channel(
        [im[:, :, 1] for im in g["blanked"]], cams, init, hull.inside_voxels(), list(g["masks"]), tuple(g["bbox"]),
        g["origin"], float(g["edge"]), tau=float(g["tau"]), alpha_l=0.006, alpha_d_eff=float(g["alpha_d_eff"]),
        max_iters=int(s["iters"]), converge_eps=1e-12, stochastic_seed=0, g_sigma=float(s["g_sigma"]))
    assert np.array_equal(np.array(rmse), s["rmse_seed0"])
    assert np.array_equal(vals, s["green_seed0"])
