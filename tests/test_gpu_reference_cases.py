"""The reference's own known-answer tests (pkg/tests/test_render.py,
test_reconstruct.py, test_radiometry.py) run through the device path."""

import numpy as np
import pytest

from paper_1809_06417_b200 import (
    Camera,
    FlameMask,
    HullTags,
    ReconstructionConfig,
    RenderConfig,
    VoxelGrid,
    adjust_pass,
    build_color_temp_map,
    look_at,
    render_pixels,
    render_view,
    temp_from_green,
)
from paper_1809_06417_b200.volume import OUTSIDE_HULL

pytestmark = pytest.mark.gpu


def ring_camera(azimuth_deg, radius=0.3, width=80, height=60, fov_deg=60.0):
    a = np.radians(azimuth_deg)
    R, t = look_at(radius * np.array([np.cos(a), np.sin(a), 0.0]), (0.0, 0.0, 0.0))
    f = (height / 2.0) / np.tan(np.radians(fov_deg) / 2.0)
    return Camera(fx=f, fy=f, cx=width / 2.0, cy=height / 2.0, rotation=R, translation=t, width=width, height=height)


def const_grid(n, value, edge=None, tag="red"):
    edge = edge if edge is not None else 0.2 / n
    return VoxelGrid(n, n, n, np.array([-0.5 * n * edge] * 3), edge, tag,
                     np.full((n + 1,) * 3, value, dtype=np.float32))


def axis_camera(grid, width=1, height=1):
    """A 1-pixel camera whose single ray is the x axis through (0, -0.001, -0.001)."""
    R, t = look_at((grid.origin[0] - 1.0, -0.001, -0.001), (0.0, -0.001, -0.001), up=(0.0, 0.0, 1.0))
    return Camera(fx=10.0, fy=10.0, cx=0.5, cy=0.5, rotation=R, translation=t, width=width, height=height)


def test_single_sample_hand_value(cuda_device):
    g = const_grid(1, 100.0, edge=0.2)
    out = render_pixels(axis_camera(g), [g], RenderConfig(), np.array([0.5]), np.array([0.5]))
    assert out[0, 0] == pytest.approx(5.0, rel=1e-6)


@pytest.mark.parametrize("n,emission,bg", [(8, 100.0, 0.0), (64, 37.5, 12.0), (21, 200.0, 3.0)])
def test_geometric_closed_form(cuda_device, n, emission, bg):
    g = const_grid(n, emission)
    cfg = RenderConfig(background=np.array([bg] * 3))
    out = render_pixels(axis_camera(g), [g], cfg, np.array([0.5]), np.array([0.5]))
    tau = cfg.tau
    closed = emission * (1 - (1 - tau) ** n) + (1 - tau) ** n * bg
    assert out[0, 0] == pytest.approx(closed, rel=1e-6)


@pytest.mark.parametrize("scattering", [False, True])
def test_sentinel_clamps_to_zero(cuda_device, scattering):
    g = VoxelGrid(8, 8, 8, np.array([-0.1] * 3), 0.025, "red", np.full((9, 9, 9), -1.0, np.float32))
    cfg = RenderConfig(scattering_enabled=scattering, sigma_s=0.3)
    img = render_view(ring_camera(30.0), [g], None, cfg)
    assert np.all(img.data == 0.0)


def test_empty_volume_is_background(cuda_device):
    g = const_grid(8, 0.0)
    img = render_view(ring_camera(30.0), [g, g.copy("green"), g.copy("blue")], None,
                      RenderConfig(background=np.array([7.0, 8.0, 9.0])))
    assert img.data.shape == (60, 80, 3)
    assert img.data[:, :, 0].max() <= 7.0 + 1e-5
    assert np.allclose(img.data[0, 0], [7.0, 8.0, 9.0], atol=1e-5)


def test_linearity_and_monotonicity(cuda_device):
    rng = np.random.default_rng(3)
    vals = rng.uniform(0, 100, size=(9, 9, 9)).astype(np.float32)
    g1 = VoxelGrid(8, 8, 8, np.array([-0.1] * 3), 0.025, "red", vals)
    g2 = VoxelGrid(8, 8, 8, np.array([-0.1] * 3), 0.025, "red", 2.0 * vals)
    cam = ring_camera(17.0)
    for scattering in (False, True):
        cfg = RenderConfig(scattering_enabled=scattering, sigma_s=0.2)
        a = render_view(cam, [g1], None, cfg).data.astype(np.float64)
        b = render_view(cam, [g2], None, cfg).data.astype(np.float64)
        assert np.allclose(b, 2.0 * a, rtol=1e-5, atol=1e-4)
        bumped = g1.copy()
        bumped.values[4, 4, 4] += 10.0
        c = render_view(cam, [bumped], None, cfg).data
        assert np.all(c >= render_view(cam, [g1], None, cfg).data - 1e-5)


def test_scattering_only_adds_light(cuda_device):
    g = const_grid(8, 60.0)
    cam = ring_camera(45.0)
    base = render_view(cam, [g], None, RenderConfig()).data.sum()
    for dirs in (8, 32):
        img = render_view(cam, [g], None, RenderConfig(sigma_s=0.3, scattering_enabled=True, scatter_dirs=dirs))
        assert img.data.sum() > base


# --- adjust_pass (reference tests/test_reconstruct.py:153-250) -----------------


def face_on_camera(width=9, height=9, dist=1.0):
    R, t = look_at((0.0, 0.0, -dist), (0.0, 0.0, 0.0), up=(0.0, 1.0, 0.0))
    return Camera(fx=18.0, fy=18.0, cx=width / 2.0, cy=height / 2.0, rotation=R, translation=t,
                  width=width, height=height)


def full_mask(cam):
    return FlameMask(cam.width, cam.height, np.ones((cam.height, cam.width), bool))


def test_adjust_zero_residual_is_identity(cuda_device):
    cam = face_on_camera()
    grid = VoxelGrid(4, 4, 4, np.array([-0.2] * 3), 0.1, "red",
                     np.random.default_rng(0).uniform(0, 50, (5, 5, 5)).astype(np.float32))
    before = grid.values.copy()
    adjust_pass(grid, HullTags(np.ones((4, 4, 4), np.uint32), 1), [cam], [np.zeros((9, 9))], [full_mask(cam)],
                ReconstructionConfig(deterministic_mode=True), np.random.default_rng(0))
    assert np.array_equal(grid.values, before)


def test_adjust_single_sample_hand_trace(cuda_device):
    edge = 0.1
    grid = VoxelGrid(1, 1, 1, np.array([-edge / 2] * 3), edge, "red")
    R, t = look_at((0.0, 0.0, -1.0), (0.0, 0.0, 0.0), up=(0, 1, 0))
    cam = Camera(fx=40.0, fy=40.0, cx=0.5, cy=0.5, width=1, height=1, rotation=R, translation=t)
    cfg = ReconstructionConfig(alpha_l=0.001, alpha_d=1.0, deterministic_mode=True)
    adjust_pass(grid, HullTags(np.ones((1, 1, 1), np.uint32), 1), [cam], [np.full((1, 1), 100.0)],
                [full_mask(cam)], cfg, np.random.default_rng(0))
    expected = 0.001 * 100.0 * np.exp(-cfg.effective_alpha_d(grid) * np.sqrt(3) * edge / 2)
    assert np.allclose(grid.values, expected, rtol=1e-6)


def test_adjust_preserves_sentinel_and_sign(cuda_device):
    cam = face_on_camera()
    tags = np.zeros((4, 4, 4), np.uint32)
    tags[1:3, 1:3, 1:3] = 1
    hull = HullTags(tags, 1)
    kp = hull.key_point_mask()
    grid = VoxelGrid(4, 4, 4, np.array([-0.2] * 3), 0.1, "red",
                     np.where(kp, np.float32(0.0), np.float32(OUTSIDE_HULL)))
    adjust_pass(grid, hull, [cam], [np.full((9, 9), 50.0)], [full_mask(cam)],
                ReconstructionConfig(deterministic_mode=True), np.random.default_rng(0))
    assert np.all(grid.values[~kp] == OUTSIDE_HULL)
    assert np.any(grid.values[kp] > 0.0)
    full = HullTags(np.ones((4, 4, 4), np.uint32), 1)
    g2 = VoxelGrid(4, 4, 4, np.array([-0.2] * 3), 0.1, "red")
    adjust_pass(g2, full, [cam], [np.full((9, 9), 25.0)], [full_mask(cam)],
                ReconstructionConfig(deterministic_mode=True), np.random.default_rng(0))
    assert np.all(g2.values > 0.0)


def test_adjust_respects_flame_mask(cuda_device):
    cam = face_on_camera()
    g = VoxelGrid(4, 4, 4, np.array([-0.2] * 3), 0.1, "red")
    adjust_pass(g, HullTags(np.ones((4, 4, 4), np.uint32), 1), [cam], [np.full((9, 9), 25.0)],
                [FlameMask(9, 9, np.zeros((9, 9), bool))], ReconstructionConfig(deterministic_mode=True),
                np.random.default_rng(0))
    assert np.all(g.values == 0.0)


def test_adjust_stochastic_seed_reproducible(cuda_device):
    cam = face_on_camera()
    hull = HullTags(np.ones((4, 4, 4), np.uint32), 1)
    outs = []
    for seed in (7, 7, 8):
        g = VoxelGrid(4, 4, 4, np.array([-0.2] * 3), 0.1, "red")
        adjust_pass(g, hull, [cam], [np.full((9, 9), 25.0)], [full_mask(cam)], ReconstructionConfig(g_sigma=0.1),
                    np.random.default_rng(seed))
        outs.append(g.values.copy())
    assert np.array_equal(outs[0], outs[1])
    assert not np.array_equal(outs[0], outs[2])


# --- radiometry (reference tests/test_radiometry.py:67-106) --------------------


def test_temperature_map_endpoints_and_clamps(cuda_device):
    cmap = build_color_temp_map(1000.0, 2300.0, 1.0)
    assert cmap.entries.max() == 255.0
    assert np.all(np.diff(cmap.green) > 0)
    t, c = temp_from_green(cmap, cmap.green[0])
    assert t == pytest.approx(cmap.t_min) and not c
    t, c = temp_from_green(cmap, cmap.green[-1])
    assert t == pytest.approx(cmap.t_max) and not c
    t, c = temp_from_green(cmap, cmap.green[-1] * 2.0)
    assert c and t == cmap.t_max
    t, c = temp_from_green(cmap, -1.0)
    assert c and t == cmap.t_min
    rng = np.random.default_rng(42)
    temps = rng.uniform(cmap.t_min, cmap.t_max, size=50)
    back, clamped = temp_from_green(cmap, cmap.green_of(temps))
    assert not clamped.any() and np.all(np.abs(back - temps) <= cmap.step)
    with pytest.raises(ValueError):
        build_color_temp_map(2300.0, 1000.0, 1.0)


def test_render_views_batch_equals_render_view(cuda_device):
    """The batched renderer (one launch, 8x4 warp patches) is bit-identical to
    per-view render_view: skipped samples add exactly 0 whatever the warp."""
    from paper_1809_06417_b200 import render_views
    from paper_1809_06417_b200.synth import synth_cameras, synth_volume

    vols = synth_volume((24, 24, 24), seed=3, kind="flame")
    grids = [vols[t] for t in ("red", "green", "blue")]
    cams = synth_cameras(3, elevation_jitter_deg=5.0, width=96, height=64, seed=2)
    for cfg in (RenderConfig(), RenderConfig(scattering_enabled=True, sigma_s=0.1)):
        batch = render_views(cams, grids, cfg)
        for cam, img in zip(cams, batch):
            assert np.array_equal(img.data, render_view(cam, grids, None, cfg).data)
