"""Host-side API of the drop-in (no GPU): the reference's known-answer tests
for the scalar fp64 forms, geometry, preprocessing, configs, trace CSV, and
the view-sharding arithmetic.  Mirrors /root/reference/pkg/tests/
test_render.py, test_reconstruct.py, test_geometry.py, test_volume.py."""

import numpy as np
import pytest

from paper_1809_06417_b200 import (
    Camera,
    EmptyHullError,
    HullTags,
    Image,
    IterationTrace,
    NoFlameError,
    PhaseConfig,
    Ray,
    ReconstructionConfig,
    RenderConfig,
    VoxelGrid,
    adjustment_value,
    bounding_box,
    in_scatter,
    integrate_ray,
    look_at,
    march,
    pixel_ray,
    pixel_rays,
    project,
    rmse_pixels,
    rmse_volume,
    sample_transparency,
    sample_trilinear,
    threshold_mask,
    write_trace_csv,
)
from paper_1809_06417_b200.engine import shard_views
from paper_1809_06417_b200.preprocess import FlameMask, Rect


def const_grid(n, value, edge=None, tag="red"):
    edge = edge if edge is not None else 0.2 / n
    vals = np.full((n + 1, n + 1, n + 1), value, dtype=np.float32)
    return VoxelGrid(n, n, n, np.array([-0.5 * n * edge] * 3), edge, tag, vals)


def axis_ray(grid):
    return Ray(np.array([grid.origin[0] - 1.0, -0.001, -0.001]), np.array([1.0, 0.0, 0.0]))


# --- render (scalar forms) -----------------------------------------------------


def test_march_axis_aligned_count_and_first_sample():
    g = const_grid(64, 1.0)
    s = march(axis_ray(g), g)
    assert len(s) == 64 and [p.order_k for p in s] == list(range(1, 65))
    assert s[0].position[0] == pytest.approx(g.origin[0] + 0.5 * g.edge, abs=1e-12)


def test_march_miss_is_empty():
    g = const_grid(8, 1.0)
    assert march(Ray(np.array([10.0, 10.0, 10.0]), np.array([0.0, 0.0, 1.0])), g) == []


def test_accumulated_transparency_is_exact():
    for k in (1, 2, 7, 16, 33, 64):
        g = const_grid(k, 0.0, edge=0.01)
        cfg = RenderConfig(background=np.array([1.0, 1.0, 1.0]))
        assert integrate_ray(axis_ray(g), [g], None, cfg)[0] == sample_transparency(k + 1, cfg.tau)


def test_single_sample_hand_value():
    g = const_grid(1, 100.0, edge=0.2)
    assert integrate_ray(axis_ray(g), [g], None, RenderConfig())[0] == pytest.approx(5.0, rel=1e-12)


@pytest.mark.parametrize("n,emission,bg", [(8, 100.0, 0.0), (64, 37.5, 12.0), (21, 200.0, 3.0)])
def test_geometric_closed_form(n, emission, bg):
    g = const_grid(n, emission)
    cfg = RenderConfig(background=np.array([bg] * 3))
    tau = cfg.tau
    closed = emission * (1 - (1 - tau) ** n) + (1 - tau) ** n * bg
    assert integrate_ray(axis_ray(g), [g], None, cfg)[0] == pytest.approx(closed, rel=1e-6)


def test_sentinel_clamps_to_zero():
    g = VoxelGrid(8, 8, 8, np.array([-0.1] * 3), 0.025, "red", np.full((9, 9, 9), -1.0, np.float32))
    assert integrate_ray(axis_ray(g), [g], None, RenderConfig())[0] == 0.0


def test_in_scatter_uniform_isotropic():
    g = const_grid(16, 80.0)
    cfg = RenderConfig(sigma_s=1.0, scattering_enabled=True, scatter_dirs=64)
    assert in_scatter([g], g.origin + g.box.size / 2, cfg, PhaseConfig(0.0))[0] == pytest.approx(80.0, rel=1e-2)


def test_render_config_validation():
    for kw in ({"tau": 0.0}, {"tau": 1.0}, {"sigma_a": -0.1}, {"scattering_enabled": True, "scatter_dirs": 0}):
        with pytest.raises(ValueError):
            RenderConfig(**kw)


# --- geometry / volume ---------------------------------------------------------


def test_pixel_ray_off_axis_direction():
    cam = Camera(fx=500.0, fy=500.0, cx=320.0, cy=240.0, rotation=np.eye(3), translation=np.zeros(3),
                 width=640, height=480)
    r = pixel_ray(cam, 420.0, 240.0)
    d = np.array([100.0 / 500.0, 0.0, 1.0])
    assert np.allclose(r.direction, d / np.linalg.norm(d), atol=1e-12)
    o, dirs = pixel_rays(cam, np.array([420.0]), np.array([240.0]))
    assert np.allclose(dirs[0], r.direction, atol=1e-15)


def test_project_round_trip():
    R, t = look_at((0.3, 0.1, 0.05), (0.0, 0.0, 0.0))
    cam = Camera(fx=400.0, fy=400.0, cx=160.0, cy=120.0, rotation=R, translation=t, width=320, height=240)
    u, v, z = project(cam, np.array([0.01, -0.02, 0.03]))
    ray = pixel_ray(cam, u, v)
    p = ray.at(np.linalg.norm(cam.center - np.array([0.01, -0.02, 0.03])))
    assert np.allclose(p, [0.01, -0.02, 0.03], atol=1e-9)


def test_camera_validation():
    with pytest.raises(ValueError):
        Camera(fx=-1.0, fy=1.0, cx=1.0, cy=1.0, rotation=np.eye(3), translation=np.zeros(3), width=4, height=4)
    with pytest.raises(ValueError):
        Camera(fx=1.0, fy=1.0, cx=1.0, cy=1.0, rotation=np.diag([1.0, 1.0, -1.0]), translation=np.zeros(3),
               width=4, height=4)


def test_trilinear_matches_weight_oracle():
    rng = np.random.default_rng(1)
    vals = rng.uniform(0, 10, (5, 5, 5)).astype(np.float32)
    g = VoxelGrid(4, 4, 4, np.zeros(3), 0.5, "red", vals)
    p = np.array([0.7, 1.3, 0.2])
    q = p / 0.5
    i = np.floor(q).astype(int)
    f = q - i
    ref = 0.0
    for dx in (0, 1):
        for dy in (0, 1):
            for dz in (0, 1):
                w = (f[0] if dx else 1 - f[0]) * (f[1] if dy else 1 - f[1]) * (f[2] if dz else 1 - f[2])
                ref += w * vals[i[0] + dx, i[1] + dy, i[2] + dz]
    assert sample_trilinear(g, p) == pytest.approx(ref, rel=1e-12)


def test_key_point_mask_dilates_inside_voxels():
    tags = np.zeros((4, 4, 4), np.uint32)
    tags[1, 2, 3] = 3
    tags[0, 0, 0] = 1  # not inside: only one of two views
    kp = HullTags(tags, 2).key_point_mask()
    assert kp.sum() == 8 and kp[1:3, 2:4, 3:5].all()
    with pytest.raises(ValueError):
        HullTags(np.full((2, 2, 2), 4, np.uint32), 2)


# --- preprocess ----------------------------------------------------------------


def test_threshold_mask_and_bbox():
    data = np.zeros((20, 30, 3), np.float32)
    data[5, 7] = [0.0, 31.0, 0.0]
    data[12, 20] = [30.0, 30.0, 30.0]  # not strictly above
    m, blanked = threshold_mask(Image(30, 20, 3, data))
    assert m.count == 1 and blanked.data[12, 20].sum() == 0
    assert bounding_box([m], 4) == Rect(3, 1, 11, 9)
    with pytest.raises(NoFlameError):
        bounding_box([FlameMask(30, 20, np.zeros((20, 30), bool))])


# --- reconstruct helpers -------------------------------------------------------


def test_adjustment_value_hand_case():
    cfg = ReconstructionConfig(alpha_l=0.001, alpha_d=1.0, tau=0.05)
    assert adjustment_value(100.0, 1, 0.0, cfg) == pytest.approx(0.1, rel=1e-12)
    with pytest.raises(ValueError):
        adjustment_value(1.0, 0, 0.0, cfg)


def test_rmse_helpers():
    a = Image(8, 8, 3, np.full((8, 8, 3), 10.0, np.float32))
    b = Image(8, 8, 3, np.full((8, 8, 3), 13.0, np.float32))
    assert np.allclose(rmse_pixels(a, b, Rect(0, 0, 7, 7)), 3.0)
    tags = np.zeros((2, 2, 2), np.uint32)
    tags[0, 0, 0] = 1
    g1 = VoxelGrid(2, 2, 2, np.zeros(3), 0.1, "red")
    g3 = g1.copy()
    g3.values[0, 0, 0] = 8.0
    assert rmse_volume(g1, g3, HullTags(tags, 1)) == pytest.approx(np.sqrt(64.0 / 8.0))
    with pytest.raises(EmptyHullError):
        rmse_volume(g1, g1, HullTags(np.zeros((2, 2, 2), np.uint32), 1))


def test_reconstruction_config_validation_and_alpha_scaling():
    for kw in ({"alpha_l": 0.0}, {"tau": 1.5}, {"converge_eps": 0.0}, {"max_iters": 0}, {"g_sigma": -1.0}):
        with pytest.raises(ValueError):
            ReconstructionConfig(**kw)
    g = VoxelGrid(10, 10, 10, np.zeros(3), 0.04)
    assert ReconstructionConfig(alpha_d=2.0).effective_alpha_d(g) == pytest.approx(2.0 * 0.2 / 0.4)


def test_trace_csv(tmp_path):
    traces = {
        "red": IterationTrace(rmse=[5.0, 3.0], wall_ms=[10.0, 11.0], converged=True),
        "green": IterationTrace(rmse=[4.0, 2.0, 1.0], wall_ms=[9.0, 9.0, 9.0], vol_rmse=[40.0, 30.0, 20.0]),
        "blue": IterationTrace(rmse=[1.0], wall_ms=[8.0], converged=True),
    }
    path = tmp_path / "trace.csv"
    write_trace_csv(path, traces)
    lines = path.read_text().strip().splitlines()
    assert lines[0] == "iter,rmse_r,rmse_g,rmse_b,wall_ms,vol_rmse"
    row2 = lines[2].split(",")
    assert row2[0] == "2" and float(row2[1]) == 3.0 and float(row2[3]) == 1.0 and float(row2[4]) == 20.0


# --- multi-GPU view sharding -----------------------------------------------------


@pytest.mark.parametrize("views", [2, 3, 8, 16, 32])
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_shard_views_partition(views, world):
    ranges = [shard_views(views, r, world) for r in range(world)]
    assert ranges[0][0] == 0 and ranges[-1][1] == views
    for (a, b), (c, d) in zip(ranges, ranges[1:]):
        assert b == c
    sizes = [b - a for a, b in ranges]
    assert max(sizes) - min(sizes) <= 1
