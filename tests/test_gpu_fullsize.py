"""Parity at BASELINE config 2's full size (128^3, 8 views of 512^2, full RTE):
two device iterations against the CPU oracle on identical inputs, plus the
size-independent properties of the loop."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def scene(cuda_device):
    import bench

    return bench.make_scene()


def test_config2_two_iterations_match_oracle(scene):
    import bench
    from oracle import cpu
    from paper_1809_06417_b200 import ReconstructionConfig, reconstruct_channel
    from paper_1809_06417_b200.reconstruct import _init_grid

    sc = scene
    iters = 2
    cfg = ReconstructionConfig(alpha_l=bench.ALPHA_L, alpha_d=1.0, tau=bench.TAU, max_iters=iters,
                               converge_eps=1e-12, deterministic_mode=True)
    grid, trace = reconstruct_channel(sc["images"], sc["cams"], sc["geom"], sc["hull"], cfg,
                                      render_cfg=sc["rcfg"], masks=sc["masks"], bbox=sc["bbox"])
    init = _init_grid(sc["geom"], sc["hull"], "green").values
    b = sc["bbox"]
    cpu.set_threads(0 or __import__("os").cpu_count())
    ref, ref_rmse, _, _ = cpu.reconstruct_channel(
        [im.data[:, :, 0] for im in sc["images"]], sc["cams"], init, sc["hull"].inside_voxels(),
        [m.bits for m in sc["masks"]], (b.u0, b.v0, b.u1, b.v1), sc["geom"].origin, sc["geom"].edge,
        tau=bench.TAU, scattering=True, sigma_s=bench.SIGMA_S, scatter_dirs=bench.SCAT_DIRS,
        alpha_l=bench.ALPHA_L, alpha_d_eff=cfg.effective_alpha_d(sc["geom"]), max_iters=iters,
        converge_eps=1e-12)
    np.testing.assert_allclose(trace.rmse, ref_rmse, rtol=1e-6)
    err = np.max(np.abs(grid.values.astype(np.float64) - ref) / np.maximum(np.abs(ref), 1.0))
    assert err <= 1e-4, err
    kp = sc["hull"].key_point_mask()
    assert np.all(grid.values[~kp] == -1.0)


def test_config2_loop_properties(scene):
    """Zero residual is a fixed point; results are bit-reproducible."""
    import bench
    from paper_1809_06417_b200 import ReconstructionConfig, reconstruct_channel

    sc = scene
    cfg = ReconstructionConfig(alpha_l=bench.ALPHA_L, alpha_d=1.0, tau=bench.TAU, max_iters=3,
                               converge_eps=1e-12, deterministic_mode=True)
    a, ta = reconstruct_channel(sc["images"], sc["cams"], sc["geom"], sc["hull"], cfg, render_cfg=sc["rcfg"],
                                masks=sc["masks"], bbox=sc["bbox"])
    b, tb = reconstruct_channel(sc["images"], sc["cams"], sc["geom"], sc["hull"], cfg, render_cfg=sc["rcfg"],
                                masks=sc["masks"], bbox=sc["bbox"])
    assert np.array_equal(a.values, b.values) and ta.rmse == tb.rmse
    assert ta.rmse[-1] < ta.rmse[0]
