"""Parity at BASELINE's full sizes against the CPU oracle on identical inputs
(SURVEY.md §8c contract: max |gpu - ref| / max(|ref|, 1) <= 1e-4 on the
lattice, RMSE trace to rtol 1e-6, LUT bracket indices bit-exact):

* config 2 (128^3, 8 x 512^2, full RTE): the bench's own N = 50 iterations,
  through the render plan and through the marching kernel, every iteration's
  lattice compared (reconstruct.py:250-334);
* config 3 (256^3, 16 x 1024^2, full RTE + black-body temperature):
  reconstruct_temperature for 2 iterations (reconstruct.py:415-477), the green
  lattice against the oracle and the temperatures / bracket indices
  bit-exact against numpy's interp / searchsorted on the same greens
  (radiometry.py:206-219);
* config 4 (512^3, 32 x 1024^2, full RTE): 1 iteration.

The oracle runs with its exact empty-space skip (pinned bit-identical by
tests/test_oracle_golden.py), so the whole module takes a few minutes.
profiles/r2_parity_curve_c*.json hold the per-iteration error curves from
tools/parity_curve.py."""

import numpy as np
import pytest

from tests.conftest import rel_err
from tests.fullsize_common import device_loop, loop_cfg, oracle_loop

pytestmark = pytest.mark.gpu

TOL = 1e-4


def _scene(cfg_no):
    from workloads import CONFIGS, device_scene

    return device_scene(*CONFIGS[cfg_no])


@pytest.fixture(scope="module")
def scene2(cuda_device):
    return _scene(2)


@pytest.fixture(scope="module")
def oracle2(scene2):
    return oracle_loop(scene2, 50)


@pytest.mark.parametrize("mode", ["plan", "march"])
def test_config2_fifty_iterations_match_oracle(scene2, oracle2, mode):
    ref_final, ref_rmse, ref_seen, _ = oracle2
    final, rmse, seen = device_loop(scene2, 50, mode)
    assert len(rmse) == 50 and len(seen) == 50
    np.testing.assert_allclose(rmse, ref_rmse, rtol=1e-6)
    per_iter = [rel_err(a, b) for a, b in zip(seen, ref_seen)]
    assert max(per_iter) <= TOL, per_iter
    err = rel_err(final, ref_final)
    assert err <= TOL, err
    kp = scene2["hull"].key_point_mask()
    assert np.all(final[~kp] == -1.0)


def test_config2_keypoint_order_is_bit_identical(scene2, monkeypatch):
    """Morton vs lattice numbering of the hull key points (the plans' row
    order) gives the same bits: the fixed-point sums are order-free."""
    a, ta, _ = device_loop(scene2, 3, "plan", record=False)
    monkeypatch.setenv("FVR_KP_ORDER", "lattice")
    b, tb, _ = device_loop(scene2, 3, "plan", record=False)
    assert np.array_equal(a, b) and np.array_equal(ta, tb)


def test_config2_loop_properties(scene2):
    """Results are bit-reproducible and the RMSE falls."""
    a, ta, _ = device_loop(scene2, 3, "plan", record=False)
    b, tb, _ = device_loop(scene2, 3, "plan", record=False)
    assert np.array_equal(a, b) and np.array_equal(ta, tb)
    assert ta[-1] < ta[0]


def test_config3_temperature_matches_oracle(cuda_device):
    import torch

    from oracle import cpu
    from paper_1809_06417_b200 import _lib, build_color_temp_map, reconstruct_temperature

    sc = _scene(3)
    iters = 2
    cmap = build_color_temp_map()
    res = reconstruct_temperature(sc["rgb"], sc["cams"], cmap, sc["geom"], loop_cfg(sc, iters),
                                  render_cfg=sc["rcfg"])
    assert res.bbox == sc["bbox"]
    assert np.array_equal(res.hull.tags, sc["hull"].tags)
    assert res.trace.iterations == iters
    ref_green, ref_rmse, _, _ = oracle_loop(sc, iters, record=False)
    np.testing.assert_allclose(res.trace.rmse, ref_rmse, rtol=1e-6)
    err = rel_err(res.green_grid.values, ref_green)
    assert err <= TOL, err

    # K-temp on the device's own greens: temperatures equal numpy's interp
    # and bracket indices equal searchsorted on numpy's table, bit for bit
    # (the device-built table is within 1e-13 of numpy's: test_gpu_parity)
    temps, green = np.ascontiguousarray(cmap.temperatures), np.ascontiguousarray(cmap.green)
    kp = sc["hull"].key_point_mask()
    g = res.green_grid.values[kp].astype(np.float64)
    T_ref, clamped = cpu.temp_from_green(green, temps, g)
    assert np.array_equal(res.temp_grid.values[kp], T_ref.astype(np.float32))
    assert np.all(res.temp_grid.values[~kp] == -1.0)
    assert res.n_clamped_low + res.n_clamped_high == int(clamped.sum())
    dev = torch.device("cuda", 0)
    vals = torch.from_numpy(np.ascontiguousarray(res.green_grid.values[kp])).to(dev)
    idx = torch.empty(vals.numel(), dtype=torch.int32, device=dev)
    out = torch.empty_like(vals)
    d_green, d_temps = torch.from_numpy(green).to(dev), torch.from_numpy(temps).to(dev)
    _lib.call("fvr_temp_lookup", vals.data_ptr(), None, vals.numel(), d_green.data_ptr(), d_temps.data_ptr(),
              green.size, out.data_ptr(), idx.data_ptr(), None, _lib.stream_ptr())
    want = cpu.bracket_index(green, g)
    got = idx.cpu().numpy()
    assert np.array_equal(out.cpu().numpy(), T_ref.astype(np.float32))
    assert np.array_equal(got, want), int((got != want).sum())


def test_config4_one_iteration_matches_oracle(cuda_device):
    sc = _scene(4)
    final, rmse, _ = device_loop(sc, 1, "plan", record=False)
    ref_final, ref_rmse, _, _ = oracle_loop(sc, 1, record=False)
    np.testing.assert_allclose(rmse, ref_rmse, rtol=1e-6)
    err = rel_err(final, ref_final)
    assert err <= TOL, err
