"""The wide (8-byte) plan entries: render-plan columns for hulls of >= 2^24
key points and adjust-plan residual indices for V * P >= 2^24 -- the sizes
where the 24-bit fields of the 6-byte entries run out.  The reference has no
such ceiling (volume.py:62-120), so neither may the loop: it switches to the
wide formats instead of falling back to the slower kernels.

* FVR_WIDE_PLANS=1 forces both wide formats on the golden loops: same
  parity contract against the reference's goldens, and the 17-bit-mantissa
  narrow plans agree with the f32-weight wide ones to 1e-5;
* a 288^3 lattice whose hull fills most of the box has ~21 M > 2^24 key
  points: the loop picks the wide render plan by itself and matches the CPU
  oracle after one iteration."""

import numpy as np
import pytest

from tests.conftest import load_golden, rel_err

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("fixture", ["config1.npz", "loop_scatter.npz"])
def test_forced_wide_plans_match_reference(cuda_device, fixture, monkeypatch):
    from paper_1809_06417_b200 import ReconstructionConfig, reconstruct_channel
    from tests.test_gpu_parity import _loop_inputs

    g = load_golden(fixture)
    cams, hull, images, masks, bbox, geom, rcfg = _loop_inputs(g)
    cfg = ReconstructionConfig(alpha_l=0.006, alpha_d=1.0, tau=float(g["tau"]), max_iters=int(g["iters"]),
                               converge_eps=1e-12, deterministic_mode=True)
    narrow, tn = reconstruct_channel(images, cams, geom, hull, cfg, render_cfg=rcfg, masks=masks, bbox=bbox)
    monkeypatch.setenv("FVR_WIDE_PLANS", "1")
    wide, tw = reconstruct_channel(images, cams, geom, hull, cfg, render_cfg=rcfg, masks=masks, bbox=bbox)
    np.testing.assert_allclose(tw.rmse, g["rmse"], rtol=1e-6)
    assert rel_err(wide.values, g["green"]) <= 1e-4
    assert rel_err(wide.values, narrow.values) <= 1e-5
    np.testing.assert_allclose(tw.rmse, tn.rmse, rtol=1e-6)


def test_hull_beyond_24_bits_uses_wide_render_plan(cuda_device):
    import torch

    from paper_1809_06417_b200 import (
        HullTags, RenderConfig, ReconstructionConfig, VoxelGrid, compute_visual_hull, reconstruct_channel, render_view,
    )
    from paper_1809_06417_b200.engine import ChannelLoop
    from paper_1809_06417_b200.preprocess import bounding_box, threshold_mask
    from paper_1809_06417_b200.reconstruct import _init_grid, _loop_config
    from paper_1809_06417_b200.synth import synth_cameras, synth_volume
    from tests.fullsize_common import oracle_loop

    n = 288
    vols = synth_volume((n, n, n), seed=0, kind="slab", slab_value=60.0)
    truth = [vols[t] for t in ("red", "green", "blue")]
    cams = synth_cameras(2, radius=0.6, fov=40.0, width=48, height=48, seed=0)
    tau = 1.0 - 0.95 ** (64.0 / n)
    rcfg = RenderConfig(tau=tau, scattering_enabled=True, sigma_s=0.1, scatter_dirs=32)
    imgs = [render_view(c, truth, None, rcfg) for c in cams]
    masked = [threshold_mask(im) for im in imgs]
    masks = [m for m, _ in masked]
    bbox = bounding_box(masks, 4)
    geom = VoxelGrid(n, n, n, truth[0].origin, truth[0].edge)
    hull = compute_visual_hull(geom, [m.bits for m in masks], cams)
    assert isinstance(hull, HullTags)
    kp = hull.key_point_mask()
    assert int(kp.sum()) >= 1 << 24, int(kp.sum())
    images = [im.channel(1) for _, im in masked]
    cfg = ReconstructionConfig(alpha_l=0.006, alpha_d=1.0, tau=tau, max_iters=1, converge_eps=1e-12,
                               deterministic_mode=True)
    grid0 = _init_grid(geom, hull, "green")
    loop = ChannelLoop(cams, grid0, grid0.values, [im.data[bbox.slices][:, :, 0] for im in images], masks, bbox,
                       hull.inside_voxels(), kp, rcfg, _loop_config(cfg, grid0), 1, use_graph=False)
    assert loop.rplan and loop.rp_wide, (loop.rplan, getattr(loop, "rp_wide", None))
    del loop
    torch.cuda.empty_cache()
    grid, trace = reconstruct_channel(images, cams, geom, hull, cfg, render_cfg=rcfg, masks=masks, bbox=bbox)
    sc = dict(n=n, tau=tau, images=images, cams=cams, hull=hull, masks=masks, bbox=bbox, geom=geom, rcfg=rcfg)
    ref, ref_rmse, _, _ = oracle_loop(sc, 1, record=False)
    np.testing.assert_allclose(trace.rmse, ref_rmse, rtol=1e-6)
    assert rel_err(grid.values, ref) <= 1e-4
