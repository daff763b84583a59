"""GPU parity: the sm_100a path against the reference's golden vectors and
the CPU oracle, through the C ABI (paper_1809_06417_b200._kernels shims and
the public API).  Tolerance: max |gpu - ref| / max(|ref|, 1)
<= 1e-4 on pixels and key points; integer outputs exact."""

import numpy as np
import pytest

from oracle import cpu
from paper_1809_06417_b200 import (
    Camera,
    HullTags,
    Image,
    ReconstructionConfig,
    RenderConfig,
    VoxelGrid,
    _kernels,
    build_color_temp_map,
    compute_visual_hull,
    reconstruct_channel,
    reconstruct_color,
    render_view,
    temp_from_green,
)
from paper_1809_06417_b200 import _lib
from paper_1809_06417_b200.preprocess import FlameMask, Rect
from paper_1809_06417_b200.radiometry import ColorTempMap, fibonacci_sphere
from tests.conftest import cameras_from, load_golden, rel_err

pytestmark = pytest.mark.gpu
TOL = 1e-4


@pytest.fixture(scope="module")
def kern(cuda_device):
    return load_golden("kernels.npz")


@pytest.mark.parametrize("name,scat,sig,g,nd", [("plain", False, 0.0, 0.0, 1),
                                                ("scat", True, 0.3, 0.0, 32),
                                                ("scat_g", True, 0.3, 0.4, 16)])
def test_render_rays(kern, name, scat, sig, g, nd):
    out = np.empty((kern["dirs"].shape[0], 2))
    sd = fibonacci_sphere(nd) if scat else np.zeros((1, 3))
    _kernels.render_rays(kern["origin"], kern["dirs"], kern["values"], kern["lo"], float(kern["edge"]), 0.05, 1.0,
                         kern["background"], scat, sig, sd, g, float(kern["edge"]), out)
    assert rel_err(out, kern["render_" + name]) <= TOL


def test_render_rays_inner_origin(kern):
    out = np.empty((kern["dirs"].shape[0], 2))
    _kernels.render_rays(kern["inner"], kern["dirs"], kern["values"], kern["lo"], float(kern["edge"]), 0.05, 1.0,
                         kern["background"], False, 0.0, np.zeros((1, 3)), 0.0, float(kern["edge"]), out)
    assert rel_err(out, kern["render_inner"]) <= TOL


def test_count_hull_samples_exact(kern):
    counts = np.empty(kern["dirs"].shape[0], dtype=np.int64)
    _kernels.count_hull_samples(kern["origin"], kern["dirs"], kern["inside"], kern["lo"], float(kern["edge"]), counts)
    assert np.array_equal(counts, kern["counts"])


@pytest.mark.parametrize("use_g", [False, True])
def test_adjust_rays(kern, use_g):
    n = int(kern["n"])
    parts = np.zeros((16, n + 1, n + 1, n + 1))
    gv = kern["g_values"] if use_g else np.ones(1)
    go = kern["g_offsets"] if use_g else np.zeros(kern["dirs"].shape[0], np.int64)
    _kernels.adjust_rays_chunked(kern["origin"], kern["dirs"], kern["residuals"], gv, go, use_g, kern["inside"],
                                 kern["lo"], float(kern["edge"]), 0.05, 0.006, 1.0, parts)
    ref = kern["adjust_g" if use_g else "adjust_det"]
    got = parts.sum(axis=0)
    assert np.max(np.abs(got - ref)) <= 1e-5 * max(1.0, np.abs(ref).max())
    assert np.array_equal(got != 0, ref != 0)  # same key points touched: exact cells


def _render_grids(g):
    return [VoxelGrid(16, 16, 16, g["origin"], float(g["edge"]), t, g["values"][i])
            for i, t in enumerate(("red", "green", "blue"))]


def test_render_view_rgb(cuda_device):
    g = load_golden("render.npz")
    cam = cameras_from(g, Camera)[0]
    grids = _render_grids(g)
    img = render_view(cam, grids, None, RenderConfig(background=np.array([1.0, 2.0, 3.0])))
    assert rel_err(img.data, g["plain"]) <= TOL
    single = render_view(cam, [grids[1]], None, RenderConfig(background=np.array([1.0, 2.0, 3.0])))
    assert rel_err(single.data, g["single_green"]) <= TOL


def test_render_view_scattering(cuda_device):
    g = load_golden("render.npz")
    cam = cameras_from(g, Camera)[0]
    img = render_view(cam, _render_grids(g), None, RenderConfig(sigma_s=0.3, scattering_enabled=True, scatter_dirs=32))
    assert rel_err(img.data, g["scat"]) <= TOL


def _loop_inputs(g):
    cams = cameras_from(g, Camera)
    n = int(g["n"])
    hull = HullTags(g["hull_tags"], len(cams))
    images = [Image(im.shape[1], im.shape[0], 1, im[:, :, 1:2]) for im in g["blanked"]]
    masks = [FlameMask(m.shape[1], m.shape[0], m) for m in g["masks"]]
    u0, v0, u1, v1 = (int(x) for x in g["bbox"])
    geom = VoxelGrid(n, n, n, g["origin"], float(g["edge"]))
    rcfg = RenderConfig(tau=float(g["tau"]), scattering_enabled=bool(g["scattering"]), sigma_s=float(g["sigma_s"]))
    return cams, hull, images, masks, Rect(u0, v0, u1, v1), geom, rcfg


@pytest.mark.parametrize("fixture", ["config1.npz", "loop_scatter.npz"])
def test_reconstruct_channel_parity(cuda_device, fixture):
    g = load_golden(fixture)
    cams, hull, images, masks, bbox, geom, rcfg = _loop_inputs(g)
    cfg = ReconstructionConfig(alpha_l=0.006, alpha_d=1.0, tau=float(g["tau"]), max_iters=int(g["iters"]),
                               converge_eps=1e-12, deterministic_mode=True)
    grid, trace = reconstruct_channel(images, cams, geom, hull, cfg, render_cfg=rcfg, masks=masks, bbox=bbox,
                                      tag="green")
    assert trace.iterations == int(g["iters"])
    assert trace.converged == bool(g["converged"])
    np.testing.assert_allclose(trace.rmse, g["rmse"], rtol=1e-6)
    assert rel_err(grid.values, g["green"]) <= TOL
    kp = hull.key_point_mask()
    assert np.all(grid.values[~kp] == -1.0)


def test_reconstruct_run_to_run_bit_identical(cuda_device):
    g = load_golden("config1.npz")
    cams, hull, images, masks, bbox, geom, rcfg = _loop_inputs(g)
    cfg = ReconstructionConfig(alpha_l=0.006, tau=0.05, max_iters=6, converge_eps=1e-12, deterministic_mode=True)
    a, ta = reconstruct_channel(images, cams, geom, hull, cfg, render_cfg=rcfg, masks=masks, bbox=bbox)
    b, tb = reconstruct_channel(images, cams, geom, hull, cfg, render_cfg=rcfg, masks=masks, bbox=bbox)
    assert np.array_equal(a.values, b.values)
    assert ta.rmse == tb.rmse


def test_visual_hull_exact(cuda_device):
    for fixture in ("config1.npz", "loop_scatter.npz"):
        g = load_golden(fixture)
        cams = cameras_from(g, Camera)
        n = int(g["n"])
        geom = VoxelGrid(n, n, n, g["origin"], float(g["edge"]))
        hull = compute_visual_hull(geom, list(g["masks"]), cams)
        assert np.array_equal(hull.tags, g["hull_tags"])


def test_reconstruct_color_tiny_scene(cuda_device):
    g = load_golden("tiny_color.npz")
    cams = cameras_from(g, Camera)
    n = 12
    imgs = [Image(im.shape[1], im.shape[0], 3, im) for im in g["images"]]
    geom = VoxelGrid(n, n, n, np.array([-0.1] * 3), 0.2 / n)
    cfg = ReconstructionConfig(alpha_l=0.01, deterministic_mode=True, max_iters=40)
    res = reconstruct_color(imgs, cams, geom, cfg, render_cfg=RenderConfig())
    assert np.array_equal(res.hull.tags, g["hull_tags"])
    assert (res.bbox.u0, res.bbox.v0, res.bbox.u1, res.bbox.v1) == tuple(int(x) for x in g["bbox"])
    for c, tag in enumerate(("red", "green", "blue")):
        ref_rmse = g["rmse_" + tag[0]]
        assert res.traces[tag].iterations == ref_rmse.size
        np.testing.assert_allclose(res.traces[tag].rmse, ref_rmse, rtol=1e-5)
        assert rel_err(res.grids[c].values, g["grids"][c]) <= TOL


def test_color_temp_map_and_lookup(cuda_device):
    g = load_golden("ctmap.npz")
    cmap = build_color_temp_map(1000.0, 2300.0, 1.0)
    assert np.array_equal(cmap.temperatures, g["temps"])
    assert np.max(np.abs(cmap.entries - g["entries"]) / np.maximum(g["entries"], 1e-300)) <= 1e-13
    assert cmap.entries.max() == 255.0
    # every entry bit-exact (fp64 Planck in double-double, numpy's pairwise
    # trapezoid and OpenBLAS's FMA chain restated)
    assert np.array_equal(cmap.entries, g["entries"])
    odd = build_color_temp_map(1000.0, 1999.5, 3.0)
    assert np.array_equal(odd.temperatures, g["odd_temps"])
    # inversion through the reference's own table: bit-exact on every input
    ref_map = ColorTempMap(1000.0, 2300.0, 1.0, g["temps"], g["entries"])
    T, clamped = temp_from_green(ref_map, g["greens"])
    assert np.array_equal(T, g["T"])
    assert np.array_equal(clamped, g["clamped"])


def test_temp_lookup_bracket_indices_exact(cuda_device):
    t = _lib.torch()
    g = load_golden("ctmap.npz")
    green = g["entries"][:, 1]
    vals = g["greens"].astype(np.float32)
    dev = _lib.device()
    d_vals = t.from_numpy(vals).to(dev)
    d_out = t.empty_like(d_vals)
    d_idx = t.empty(vals.size, dtype=t.int32, device=dev)
    clamps = t.zeros(2, dtype=t.int64, device=dev)
    d_green = t.from_numpy(green.copy()).to(dev)
    d_temps = t.from_numpy(g["temps"].copy()).to(dev)
    _lib.call("fvr_temp_lookup", d_vals.data_ptr(), None, vals.size, d_green.data_ptr(), d_temps.data_ptr(),
              green.size, d_out.data_ptr(), d_idx.data_ptr(), clamps.data_ptr(), _lib.stream_ptr())
    idx = d_idx.cpu().numpy()
    assert np.array_equal(idx, cpu.bracket_index(green, vals.astype(np.float64)))
    T_ref, cl = cpu.temp_from_green(green, g["temps"], vals.astype(np.float64))
    assert np.array_equal(d_out.cpu().numpy(), T_ref.astype(np.float32))
    lo = int(np.sum(vals.astype(np.float64) < green[0]))
    hi = int(np.sum(vals.astype(np.float64) > green[-1]))
    assert clamps.cpu().numpy().tolist() == [lo, hi]


def test_scatter_and_gather_adjust_agree(cuda_device, monkeypatch):
    """Deterministic back-projection: the ray-driven scatter (atomics) and the
    voxel-driven gather plan both meet the reference within tolerance."""
    g = load_golden("config1.npz")
    cams, hull, images, masks, bbox, geom, rcfg = _loop_inputs(g)
    cfg = ReconstructionConfig(alpha_l=0.006, tau=0.05, max_iters=int(g["iters"]), converge_eps=1e-12,
                               deterministic_mode=True)
    monkeypatch.setenv("FVR_ADJUST", "scatter")
    a, _ = reconstruct_channel(images, cams, geom, hull, cfg, render_cfg=rcfg, masks=masks, bbox=bbox)
    monkeypatch.delenv("FVR_ADJUST")
    b, _ = reconstruct_channel(images, cams, geom, hull, cfg, render_cfg=rcfg, masks=masks, bbox=bbox)
    assert rel_err(a.values, g["green"]) <= TOL
    assert rel_err(b.values, g["green"]) <= TOL
    assert rel_err(a.values, b.values) <= 1e-5


def test_stochastic_sample_plan_matches_scatter(cuda_device, monkeypatch):
    """Stochastic mode: the sample-plan gather draws the same Philox G as the
    ray-driven scatter (same key), so the two differ only in float rounding
    order -- and the gather is bit-reproducible run to run."""
    g = load_golden("config1.npz")
    cams, hull, images, masks, bbox, geom, rcfg = _loop_inputs(g)
    cfg = ReconstructionConfig(alpha_l=0.006, tau=0.05, max_iters=8, converge_eps=1e-12, g_sigma=0.1,
                               rng_seed=11, deterministic_mode=False)
    monkeypatch.setenv("FVR_ADJUST", "scatter")
    a, ta = reconstruct_channel(images, cams, geom, hull, cfg, render_cfg=rcfg, masks=masks, bbox=bbox)
    monkeypatch.delenv("FVR_ADJUST")
    b, tb = reconstruct_channel(images, cams, geom, hull, cfg, render_cfg=rcfg, masks=masks, bbox=bbox)
    c, tc = reconstruct_channel(images, cams, geom, hull, cfg, render_cfg=rcfg, masks=masks, bbox=bbox)
    assert rel_err(a.values, b.values) <= 1e-5
    np.testing.assert_allclose(ta.rmse, tb.rmse, rtol=1e-5)
    assert np.array_equal(b.values, c.values) and tb.rmse == tc.rmse
    # and the weights really are random: deterministic G gives another grid
    d, _ = reconstruct_channel(images, cams, geom, hull,
                               ReconstructionConfig(alpha_l=0.006, tau=0.05, max_iters=8, converge_eps=1e-12,
                                                    deterministic_mode=True),
                               render_cfg=rcfg, masks=masks, bbox=bbox)
    assert rel_err(b.values, d.values) > 1e-4


def test_stochastic_seed_determinism_and_grayscale(cuda_device):
    """tests/test_reconstruct.py:311-341 of the reference: equal seeds give
    identical grids and traces, different seeds differ, and grayscale input
    yields three bit-equal channels (each channel restarts the stream)."""
    g = load_golden("tiny_color.npz")
    cams = cameras_from(g, Camera)
    imgs = [Image(im.shape[1], im.shape[0], 3, im) for im in g["images"]]
    geom = VoxelGrid(12, 12, 12, np.array([-0.1] * 3), 0.2 / 12)
    outs = []
    for seed in (3, 3, 4):
        cfg = ReconstructionConfig(alpha_l=0.01, max_iters=5, g_sigma=0.1, rng_seed=seed)
        outs.append(reconstruct_color(imgs, cams, geom, cfg, render_cfg=RenderConfig()))
    assert np.array_equal(outs[0].grids[0].values, outs[1].grids[0].values)
    assert outs[0].traces["red"].rmse == outs[1].traces["red"].rmse
    assert not np.array_equal(outs[0].grids[0].values, outs[2].grids[0].values)
    # grayscale images -> bit-equal channels
    gray = [Image(im.width, im.height, 3, np.repeat(im.data[:, :, 1:2], 3, axis=2)) for im in imgs]
    res = reconstruct_color(gray, cams, geom, ReconstructionConfig(alpha_l=0.01, max_iters=6, g_sigma=0.1,
                                                                   rng_seed=5), render_cfg=RenderConfig())
    assert np.array_equal(res.grids[0].values, res.grids[1].values)
    assert np.array_equal(res.grids[0].values, res.grids[2].values)


def test_empty_space_skipping_is_exact(cuda_device, monkeypatch):
    """Skipping samples whose neighbourhood is unoccupied changes nothing: the
    skipped samples add exactly 0 (the transparency still advances)."""
    g = load_golden("loop_scatter.npz")
    cams, hull, images, masks, bbox, geom, rcfg = _loop_inputs(g)
    cfg = ReconstructionConfig(alpha_l=0.006, tau=float(g["tau"]), max_iters=3, converge_eps=1e-12,
                               deterministic_mode=True)
    a, ta = reconstruct_channel(images, cams, geom, hull, cfg, render_cfg=rcfg, masks=masks, bbox=bbox)
    monkeypatch.setenv("FVR_NO_SKIP", "1")
    b, tb = reconstruct_channel(images, cams, geom, hull, cfg, render_cfg=rcfg, masks=masks, bbox=bbox)
    assert np.array_equal(a.values, b.values)
    assert ta.rmse == tb.rmse
    truth = [VoxelGrid(16, 16, 16, g["origin"], float(g["edge"]), t, g["truth"][i])
             for i, t in enumerate(("red", "green", "blue"))]
    img_noskip = render_view(cams[0], truth, None, rcfg)
    monkeypatch.delenv("FVR_NO_SKIP")
    img_skip = render_view(cams[0], truth, None, rcfg)
    assert np.array_equal(img_skip.data, img_noskip.data)
