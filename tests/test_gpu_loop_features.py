"""Loop features on the device: the NCCL exchange path (1-rank group, forced),
per-iteration callbacks, ground-truth volume RMSE, temperature snapshots,
the max-iters quirk and the convergence rule."""

import os

import numpy as np
import pytest

from paper_1809_06417_b200 import (
    Camera,
    HullTags,
    Image,
    ReconstructionConfig,
    RenderConfig,
    VoxelGrid,
    build_color_temp_map,
    reconstruct_channel,
    reconstruct_temperature,
    rmse_volume,
)
from paper_1809_06417_b200.preprocess import FlameMask, Rect
from tests.conftest import cameras_from, load_golden, rel_err

pytestmark = pytest.mark.gpu


def _inputs(name="loop_scatter.npz"):
    g = load_golden(name)
    cams = cameras_from(g, Camera)
    n = int(g["n"])
    hull = HullTags(g["hull_tags"], len(cams))
    images = [Image(im.shape[1], im.shape[0], 1, im[:, :, 1:2]) for im in g["blanked"]]
    masks = [FlameMask(m.shape[1], m.shape[0], m) for m in g["masks"]]
    u0, v0, u1, v1 = (int(x) for x in g["bbox"])
    geom = VoxelGrid(n, n, n, g["origin"], float(g["edge"]))
    rcfg = RenderConfig(tau=float(g["tau"]), scattering_enabled=bool(g["scattering"]), sigma_s=float(g["sigma_s"]))
    return g, cams, hull, images, masks, Rect(u0, v0, u1, v1), geom, rcfg


@pytest.fixture
def nccl_group(cuda_device):
    import torch.distributed as dist

    if dist.is_initialized():
        dist.destroy_process_group()
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        os.environ["MASTER_PORT"] = str(s.getsockname()[1])
    dist.init_process_group("nccl", rank=0, world_size=1)
    yield
    dist.destroy_process_group()


@pytest.mark.parametrize("stochastic", [False, True])
def test_exchange_path_matches_single_gpu(nccl_group, monkeypatch, stochastic):
    """The sharded stages (gather -> packed -> NCCL all-reduce -> finalize ->
    update_packed; scatter -> pack -> all-reduce -> unpack -> update) give the
    bit-identical grid and trace of the single-GPU stages."""
    g, cams, hull, images, masks, bbox, geom, rcfg = _inputs()
    kw = dict(alpha_l=0.006, tau=float(g["tau"]), max_iters=4, converge_eps=1e-12)
    cfg = ReconstructionConfig(g_sigma=0.1, rng_seed=3, **kw) if stochastic else \
        ReconstructionConfig(deterministic_mode=True, **kw)
    monkeypatch.setenv("FVR_NO_SHARDING", "1")
    a, ta = reconstruct_channel(images, cams, geom, hull, cfg, render_cfg=rcfg, masks=masks, bbox=bbox)
    monkeypatch.delenv("FVR_NO_SHARDING")
    monkeypatch.setenv("FVR_FORCE_SHARDED", "1")
    b, tb = reconstruct_channel(images, cams, geom, hull, cfg, render_cfg=rcfg, masks=masks, bbox=bbox)
    assert np.array_equal(a.values, b.values)
    assert ta.rmse == tb.rmse


def test_callback_and_ground_truth_trace(cuda_device):
    g, cams, hull, images, masks, bbox, geom, rcfg = _inputs()
    truth = VoxelGrid(geom.nx, geom.ny, geom.nz, geom.origin, geom.edge, "green", g["truth"][1])
    cfg = ReconstructionConfig(alpha_l=0.006, tau=float(g["tau"]), max_iters=4, converge_eps=1e-12,
                               deterministic_mode=True)
    seen = []

    def cb(it, grid, rmse):
        seen.append((it, rmse, rmse_volume(grid, truth, hull)))

    grid, trace = reconstruct_channel(images, cams, geom, hull, cfg, render_cfg=rcfg, masks=masks, bbox=bbox,
                                      ground_truth=truth, callback=cb)
    plain, ptrace = reconstruct_channel(images, cams, geom, hull, cfg, render_cfg=rcfg, masks=masks, bbox=bbox)
    assert [s[0] for s in seen] == [1, 2, 3, 4]
    assert [s[1] for s in seen] == trace.rmse == ptrace.rmse
    # device vol_rmse (pre-update grid of each iteration) matches the host metric
    np.testing.assert_allclose(trace.vol_rmse, [s[2] for s in seen], rtol=1e-9)
    assert np.array_equal(grid.values, plain.values)
    np.testing.assert_allclose(trace.rmse, g["rmse"][:4], rtol=1e-6)


def test_max_iters_quirk_and_convergence(cuda_device):
    """max_iters ends the loop after the last adjustment (the returned grid is
    one adjustment past the last RMSE); a large eps converges at iteration 2
    and returns the grid that produced the last RMSE."""
    g, cams, hull, images, masks, bbox, geom, rcfg = _inputs()
    base = dict(alpha_l=0.006, tau=float(g["tau"]), deterministic_mode=True)
    one, t1 = reconstruct_channel(images, cams, geom, hull, ReconstructionConfig(max_iters=1, converge_eps=1e-12,
                                                                                  **base),
                                  render_cfg=rcfg, masks=masks, bbox=bbox)
    two, t2 = reconstruct_channel(images, cams, geom, hull, ReconstructionConfig(max_iters=2, converge_eps=1e-12,
                                                                                  **base),
                                  render_cfg=rcfg, masks=masks, bbox=bbox)
    assert t1.iterations == 1 and not t1.converged
    assert np.any(one.values != np.where(hull.key_point_mask(), 0.0, -1.0))  # adjusted once
    conv, tc = reconstruct_channel(images, cams, geom, hull,
                                   ReconstructionConfig(max_iters=50, converge_eps=1e3, **base),
                                   render_cfg=rcfg, masks=masks, bbox=bbox)
    # rmse < eps fires at iteration 1: no adjustment at all
    assert tc.converged and tc.iterations == 1
    assert np.array_equal(conv.values, np.where(hull.key_point_mask(), np.float32(0.0), np.float32(-1.0)))
    d = abs(t2.rmse[1] - t2.rmse[0])
    conv2, tc2 = reconstruct_channel(images, cams, geom, hull,
                                     ReconstructionConfig(max_iters=50, converge_eps=d * 1.0001, **base),
                                     render_cfg=rcfg, masks=masks, bbox=bbox)
    # |rmse_2 - rmse_1| < eps fires at iteration 2: the grid is the one after one adjustment
    assert tc2.converged and tc2.iterations == 2
    assert np.array_equal(conv2.values, one.values)


def test_temperature_with_snapshots(cuda_device):
    g, cams, hull, images, masks, bbox, geom, rcfg = _inputs("config1.npz")
    rgb_imgs = [Image(im.shape[1], im.shape[0], 3, im) for im in g["images"]]
    cmap = build_color_temp_map()
    cfg = ReconstructionConfig(alpha_l=0.006, tau=0.05, max_iters=3, converge_eps=1e-12, deterministic_mode=True)
    snaps = []
    res = reconstruct_temperature(rgb_imgs, cams, cmap, geom, cfg, render_cfg=RenderConfig(),
                                  snapshot_callback=lambda it, tg, rgb: snaps.append((it, tg, rgb)))
    assert [s[0] for s in snaps] == [1, 2, 3]
    kp = res.hull.key_point_mask()
    assert np.all(res.temp_grid.values[~kp] == -1.0)
    inside = res.temp_grid.values[kp]
    assert inside.min() >= cmap.t_min and inside.max() <= cmap.t_max
    assert res.n_clamped_low + res.n_clamped_high <= kp.sum()
    # the reference's inversion of the final green grid (np.interp)
    greens = res.green_grid.values[kp].astype(np.float64)
    ref = np.interp(np.clip(greens, cmap.green[0], cmap.green[-1]), cmap.green, cmap.temperatures)
    assert np.array_equal(inside, ref.astype(np.float32))
    assert res.n_clamped_low == int(np.sum(greens < cmap.green[0]))
    assert res.n_clamped_high == int(np.sum(greens > cmap.green[-1]))
    assert len(snaps[-1][2]) == 3 and snaps[-1][2][1].channel_tag == "green"
    # every snapshot is the reference's green_to_temp + rgb_grids_from_temperature
    # (reconstruct.py:389-401, 444-455) of that iteration's green lattice, bit for bit
    greens_it = []
    reconstruct_channel([im.channel(1) for im in _blanked(rgb_imgs)], cams, geom, res.hull, cfg,
                        render_cfg=RenderConfig(), masks=res.masks if hasattr(res, "masks") else masks,
                        bbox=res.bbox, callback=lambda it, gr, r: greens_it.append(np.array(gr.values)))
    assert len(greens_it) == 3
    for (it, tg, rgb), gl in zip(snaps, greens_it):
        gk = gl[kp].astype(np.float64)
        T = np.full(gl.shape, -1.0, np.float32)
        T[kp] = np.interp(np.clip(gk, cmap.green[0], cmap.green[-1]), cmap.green, cmap.temperatures).astype(np.float32)
        assert np.array_equal(tg.values, T), it
        want = cmap.rgb_of(np.clip(T, cmap.t_min, cmap.t_max))
        for c in range(3):
            assert np.array_equal(rgb[c].values, np.where(kp, want[..., c].astype(np.float32), np.float32(-1.0))), c


def _blanked(rgb_imgs):
    from paper_1809_06417_b200.preprocess import threshold_mask

    return [threshold_mask(im)[1] for im in rgb_imgs]


def test_rgb_grids_from_temperature_matches_numpy(cuda_device):
    """Device T -> RGB (fvr_temp_rgb) against the reference's np.interp form,
    including temperatures below / above the table and exactly on nodes."""
    from paper_1809_06417_b200 import HullTags, VoxelGrid
    from paper_1809_06417_b200.reconstruct import rgb_grids_from_temperature

    cmap = build_color_temp_map()
    rng = np.random.default_rng(7)
    n = 24
    tags = (rng.random((n, n, n)) < 0.4).astype(np.uint32) * 3
    hull = HullTags(tags, 2)
    T = rng.uniform(800.0, 2500.0, (n + 1,) * 3).astype(np.float32)
    T.ravel()[:200] = cmap.temperatures[rng.integers(0, cmap.temperatures.size, 200)].astype(np.float32)
    tg = VoxelGrid(n, n, n, np.zeros(3), 0.01, "temperature", T)
    got = rgb_grids_from_temperature(tg, cmap, hull)
    kp = hull.key_point_mask()
    want = cmap.rgb_of(np.clip(T, cmap.t_min, cmap.t_max))
    for c in range(3):
        assert np.array_equal(got[c].values, np.where(kp, want[..., c].astype(np.float32), np.float32(-1.0)))


def test_rgb_batched_loop_matches_sequential(cuda_device, monkeypatch):
    """reconstruct_color's batched RGB loop (one render / gather launch for
    three channels, per-channel convergence) against three sequential
    channel loops: same iteration counts and convergence, values and traces
    within float rounding (the batched render shares stencil weights)."""
    import numpy as np

    from paper_1809_06417_b200 import Camera, Image, ReconstructionConfig, RenderConfig, VoxelGrid, reconstruct_color
    from tests.conftest import cameras_from, load_golden, rel_err

    g = load_golden("tiny_color.npz")
    cams = cameras_from(g, Camera)
    imgs = [Image(im.shape[1], im.shape[0], 3, im) for im in g["images"]]
    geom = VoxelGrid(12, 12, 12, np.array([-0.1] * 3), 0.2 / 12)
    for det in (True, False):
        cfg = ReconstructionConfig(alpha_l=0.01, deterministic_mode=det, max_iters=40, g_sigma=0.1, rng_seed=7)
        for scat in (False, True):
            rcfg = RenderConfig(scattering_enabled=scat, sigma_s=0.1 if scat else 0.0)
            monkeypatch.setenv("FVR_RGB_BATCH", "0")
            seq = reconstruct_color(imgs, cams, geom, cfg, render_cfg=rcfg)
            monkeypatch.setenv("FVR_RGB_BATCH", "1")
            bat = reconstruct_color(imgs, cams, geom, cfg, render_cfg=rcfg)
            for c, tag in enumerate(("red", "green", "blue")):
                assert bat.traces[tag].iterations == seq.traces[tag].iterations
                assert bat.traces[tag].converged == seq.traces[tag].converged
                np.testing.assert_allclose(bat.traces[tag].rmse, seq.traces[tag].rmse, rtol=1e-5)
                assert rel_err(bat.grids[c].values, seq.grids[c].values) <= 1e-5
            assert np.array_equal(bat.hull.tags, seq.hull.tags)


def test_snapshot_callbacks_stop_at_convergence_and_batch(cuda_device, monkeypatch):
    """Snapshot callbacks run off the loop's critical path (ring of pinned
    buffers): they still fire once per recorded iteration, in order, with the
    pre-update grid, none after the rule fires -- for a single channel and
    for the batched RGB loop."""
    from paper_1809_06417_b200 import reconstruct_color

    g, cams, hull, images, masks, bbox, geom, rcfg = _inputs()
    base = dict(alpha_l=0.006, tau=float(g["tau"]), deterministic_mode=True)
    _, t2 = reconstruct_channel(images, cams, geom, hull, ReconstructionConfig(max_iters=2, converge_eps=1e-12,
                                                                                **base),
                                render_cfg=rcfg, masks=masks, bbox=bbox)
    eps = abs(t2.rmse[1] - t2.rmse[0]) * 1.0001
    seen = []
    grid, tr = reconstruct_channel(images, cams, geom, hull, ReconstructionConfig(max_iters=50, converge_eps=eps,
                                                                                   **base),
                                   render_cfg=rcfg, masks=masks, bbox=bbox,
                                   callback=lambda it, gr, rmse: seen.append((it, rmse, gr.values.copy())))
    assert tr.converged and tr.iterations == 2
    assert [s[0] for s in seen] == [1, 2] and [s[1] for s in seen] == tr.rmse
    assert np.array_equal(seen[-1][2], grid.values)  # converged: the grid that produced the last RMSE

    g1 = load_golden("tiny_color.npz")
    cams1 = cameras_from(g1, Camera)
    imgs = [Image(im.shape[1], im.shape[0], 3, im) for im in g1["images"]]
    geom1 = VoxelGrid(12, 12, 12, np.array([-0.1] * 3), 0.2 / 12)
    cfg = ReconstructionConfig(alpha_l=0.01, deterministic_mode=True, max_iters=40)
    out = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("FVR_RGB_BATCH", mode)
        calls = []
        res = reconstruct_color(imgs, cams1, geom1, cfg, render_cfg=RenderConfig(),
                                callback=lambda tag, it, gr, rmse: calls.append((tag, it, rmse)))
        out[mode] = (calls, res)
    for tag in ("red", "green", "blue"):
        bat = [(it, r) for t_, it, r in out["1"][0] if t_ == tag]
        seq = [(it, r) for t_, it, r in out["0"][0] if t_ == tag]
        assert [b[0] for b in bat] == [s[0] for s in seq] == list(range(1, out["1"][1].traces[tag].iterations + 1))
        np.testing.assert_allclose([b[1] for b in bat], [s[1] for s in seq], rtol=1e-5)


@pytest.mark.parametrize("fixture,scat", [("config1.npz", False), ("loop_scatter.npz", True)])
def test_render_plan_matches_marching_render(cuda_device, monkeypatch, fixture, scat):
    """K-render through the render plan (B c + base + t_fin bg) against the
    marching kernel on the same loop: same iteration counts, traces and
    grids within float rounding -- deterministic and stochastic, one channel
    and the batched RGB loop (small grids: many samples sit within half a
    voxel of a face and take the clamped, unmerged path)."""
    from paper_1809_06417_b200 import reconstruct_color

    g = load_golden(fixture)
    cams = cameras_from(g, Camera)
    n = int(g["n"])
    hull = HullTags(g["hull_tags"], len(cams))
    images = [Image(im.shape[1], im.shape[0], 1, im[:, :, 1:2]) for im in g["blanked"]]
    masks = [FlameMask(m.shape[1], m.shape[0], m) for m in g["masks"]]
    bbox = Rect(*(int(x) for x in g["bbox"]))
    geom = VoxelGrid(n, n, n, g["origin"], float(g["edge"]))
    rcfg = RenderConfig(tau=float(g["tau"]), scattering_enabled=scat, sigma_s=float(g["sigma_s"]))
    for det in (True, False):
        cfg = ReconstructionConfig(alpha_l=0.006, tau=float(g["tau"]), max_iters=6, converge_eps=1e-12,
                                   deterministic_mode=det, g_sigma=0.1, rng_seed=1)
        monkeypatch.setenv("FVR_RENDER", "march")
        a, ta = reconstruct_channel(images, cams, geom, hull, cfg, render_cfg=rcfg, masks=masks, bbox=bbox)
        monkeypatch.setenv("FVR_RENDER", "plan")
        b, tb = reconstruct_channel(images, cams, geom, hull, cfg, render_cfg=rcfg, masks=masks, bbox=bbox)
        np.testing.assert_allclose(tb.rmse, ta.rmse, rtol=1e-6)
        assert rel_err(b.values, a.values) <= 1e-5
    rgb = [Image(im.shape[1], im.shape[0], 3, im) for im in g["images"]]
    cfg = ReconstructionConfig(alpha_l=0.006, tau=float(g["tau"]), max_iters=5, converge_eps=1e-12,
                               deterministic_mode=True)
    monkeypatch.setenv("FVR_RENDER", "march")
    a = reconstruct_color(rgb, cams, geom, cfg, render_cfg=rcfg)
    monkeypatch.setenv("FVR_RENDER", "plan")
    b = reconstruct_color(rgb, cams, geom, cfg, render_cfg=rcfg)
    for c, tag in enumerate(("red", "green", "blue")):
        np.testing.assert_allclose(b.traces[tag].rmse, a.traces[tag].rmse, rtol=1e-6)
        assert rel_err(b.grids[c].values, a.grids[c].values) <= 1e-5


@pytest.mark.gpu
@pytest.mark.parametrize("stochastic", [False, True])
def test_render_plan_layouts_and_fused_finalize(cuda_device, monkeypatch, stochastic):
    """The render plan's row order (length-sorted 16x16 tiles or natural),
    unit order (longest first or natural) and the finalize fused into its last
    CTA change only the order of float sums (and, for the fused finalize,
    nothing at all: same trace and grid bits, and the same Philox key for the
    stochastic weights)."""
    g = load_golden("config1.npz")
    cams = cameras_from(g, Camera)
    n = int(g["n"])
    hull = HullTags(g["hull_tags"], len(cams))
    images = [Image(im.shape[1], im.shape[0], 1, im[:, :, 1:2]) for im in g["blanked"]]
    masks = [FlameMask(m.shape[1], m.shape[0], m) for m in g["masks"]]
    bbox = Rect(*(int(x) for x in g["bbox"]))
    geom = VoxelGrid(n, n, n, g["origin"], float(g["edge"]))
    rcfg = RenderConfig(tau=float(g["tau"]), scattering_enabled=True, sigma_s=float(g["sigma_s"]))
    cfg = ReconstructionConfig(alpha_l=0.006, tau=float(g["tau"]), max_iters=6, converge_eps=1e-12,
                               deterministic_mode=not stochastic, g_sigma=0.1, rng_seed=5)
    monkeypatch.setenv("FVR_RENDER", "plan")

    def run(**env):
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        out = reconstruct_channel(images, cams, geom, hull, cfg, render_cfg=rcfg, masks=masks, bbox=bbox)
        for k in env:
            monkeypatch.delenv(k)
        return out

    a, ta = run()
    b, tb = run(FVR_FUSED_FINALIZE="0")
    assert ta.rmse == tb.rmse and ta.iterations == tb.iterations
    assert np.array_equal(a.values, b.values)
    for env in ({"FVR_RPLAN_TILE": "0"}, {"FVR_RPLAN_SORT": "0"}, {"FVR_RPLAN_TILE": "4x8", "FVR_RPLAN_SORT": "0"}):
        c, tc = run(**env)
        np.testing.assert_allclose(tc.rmse, ta.rmse, rtol=1e-6)
        assert rel_err(c.values, a.values) <= 1e-5


@pytest.mark.gpu
def test_render_plan_with_positive_initial_grid(cuda_device, monkeypatch):
    """An initial grid positive outside the hull: the static key points fold
    into the render plan's base (pos27 masks) and the plan still matches the
    marching kernel."""
    g = load_golden("config1.npz")
    cams = cameras_from(g, Camera)
    n = int(g["n"])
    hull = HullTags(g["hull_tags"], len(cams))
    images = [Image(im.shape[1], im.shape[0], 1, im[:, :, 1:2]) for im in g["blanked"]]
    masks = [FlameMask(m.shape[1], m.shape[0], m) for m in g["masks"]]
    bbox = Rect(*(int(x) for x in g["bbox"]))
    geom = VoxelGrid(n, n, n, g["origin"], float(g["edge"]))
    rng = np.random.default_rng(3)
    init = VoxelGrid(n, n, n, g["origin"], float(g["edge"]), "green",
                     rng.uniform(-0.5, 2.0, size=(n + 1,) * 3).astype(np.float32))
    rcfg = RenderConfig(tau=float(g["tau"]), scattering_enabled=True, sigma_s=float(g["sigma_s"]))
    cfg = ReconstructionConfig(alpha_l=0.006, tau=float(g["tau"]), max_iters=4, converge_eps=1e-12,
                               deterministic_mode=True)
    out = {}
    for mode in ("march", "plan"):
        monkeypatch.setenv("FVR_RENDER", mode)
        out[mode] = reconstruct_channel(images, cams, geom, hull, cfg, render_cfg=rcfg, masks=masks, bbox=bbox,
                                        initial=init)
    (a, ta), (b, tb) = out["march"], out["plan"]
    np.testing.assert_allclose(tb.rmse, ta.rmse, rtol=1e-6)
    assert rel_err(b.values, a.values) <= 1e-5
