"""GPU parity of the device input preparation (§8f rank 2): threshold mask,
blanked frames, union bounding box and mask summed-area tables against the
host forms of preprocess.py:59-93 / volume.py:319-324 -- all bit-exact."""

import numpy as np
import pytest

from paper_1809_06417_b200 import Camera, Image, NoFlameError, VoxelGrid, bounding_box, threshold_mask
from paper_1809_06417_b200 import _lib
from paper_1809_06417_b200.preprocess import DeviceFrames
from paper_1809_06417_b200.volume import _mask_sat, compute_visual_hull
from tests.conftest import cameras_from, load_golden

pytestmark = pytest.mark.gpu


def _frames(rng, n_views, w, h, scale=40.0):
    data = (rng.random((n_views, h, w, 3), dtype=np.float32) * scale).astype(np.float32)
    # values sitting exactly on the threshold must stay off (strict >)
    data[:, ::7, ::5, 1] = np.float32(30.0)
    return [Image(w, h, 3, d) for d in data]


@pytest.mark.parametrize("n_views,w,h,scale", [(1, 17, 9, 40.0), (4, 130, 70, 33.0), (8, 512, 512, 31.0)])
def test_device_threshold_mask_and_bbox_exact(cuda_device, n_views, w, h, scale):
    rng = np.random.default_rng(n_views * 1000 + w)
    imgs = _frames(rng, n_views, w, h, scale)
    frames = DeviceFrames(imgs)
    host = [threshold_mask(im) for im in imgs]
    for (m, b), dm, db in zip(host, frames.masks(), frames.blanked_images()):
        assert np.array_equal(m.bits, dm.bits)
        assert np.array_equal(b.data, db.data)
    ref = bounding_box([m for m, _ in host])
    assert frames.bbox == ref
    for c in range(3):
        crop = frames.channel_crops(c).cpu().numpy()
        want = np.stack([b.data[ref.slices][:, :, c] for _, b in host])
        assert np.array_equal(crop, want)


def test_device_bbox_dilation_clips_to_frame(cuda_device):
    data = np.zeros((2, 20, 30, 3), np.float32)
    data[0, 0, 29, 0] = 200.0  # corner pixel in view 0
    data[1, 19, 3, 2] = 31.0  # opposite corner in view 1
    imgs = [Image(30, 20, 3, d) for d in data]
    frames = DeviceFrames(imgs, dilate=6)
    assert frames.bbox == bounding_box([threshold_mask(im)[0] for im in imgs], dilate=6)


def test_device_frames_all_dark_raises(cuda_device):
    imgs = [Image(16, 8, 3, np.full((8, 16, 3), 30.0, np.float32)) for _ in range(3)]
    with pytest.raises(NoFlameError):
        DeviceFrames(imgs)


@pytest.mark.parametrize("w,h", [(1, 1), (13, 7), (512, 384)])
def test_mask_sat_exact(cuda_device, w, h):
    t = _lib.torch()
    rng = np.random.default_rng(w * h)
    mask = rng.random((h, w)) < 0.3
    d_mask = t.from_numpy(mask.astype(np.uint8)).to(cuda_device)
    sat = t.empty((h + 1, w + 1), dtype=t.int64, device=cuda_device)
    _lib.call("fvr_mask_sat", d_mask.data_ptr(), w, h, sat.data_ptr(), _lib.stream_ptr())
    assert np.array_equal(sat.cpu().numpy(), _mask_sat(mask))


def test_visual_hull_from_device_masks_matches_golden(cuda_device):
    t = _lib.torch()
    for fixture in ("config1.npz", "loop_scatter.npz"):
        g = load_golden(fixture)
        cams = cameras_from(g, Camera)
        n = int(g["n"])
        geom = VoxelGrid(n, n, n, g["origin"], float(g["edge"]))
        d_masks = t.from_numpy(np.stack(g["masks"]).astype(np.uint8)).to(cuda_device)
        hull = compute_visual_hull(geom, d_masks, cams)
        assert np.array_equal(hull.tags, g["hull_tags"])


def test_device_mask_ray_list_matches_host(cuda_device):
    """ChannelLoop's flame-ray list compacted on the device (torch.nonzero over
    the (V, h_bb, w_bb) masks) gives the same loop as the host list."""
    from paper_1809_06417_b200 import ReconstructionConfig, reconstruct_channel
    from paper_1809_06417_b200.preprocess import FlameMask, Rect
    from paper_1809_06417_b200.render import RenderConfig
    from paper_1809_06417_b200.volume import HullTags

    t = _lib.torch()
    g = load_golden("config1.npz")
    cams = cameras_from(g, Camera)
    n = int(g["n"])
    hull = HullTags(g["hull_tags"], len(cams))
    images = [Image(im.shape[1], im.shape[0], 1, im[:, :, 1:2]) for im in g["blanked"]]
    masks = [FlameMask(m.shape[1], m.shape[0], m) for m in g["masks"]]
    bbox = Rect(*(int(x) for x in g["bbox"]))
    geom = VoxelGrid(n, n, n, g["origin"], float(g["edge"]))
    rcfg = RenderConfig(tau=float(g["tau"]))
    cfg = ReconstructionConfig(alpha_l=0.006, tau=float(g["tau"]), max_iters=4, converge_eps=1e-12,
                               deterministic_mode=True)
    a, ta = reconstruct_channel(images, cams, geom, hull, cfg, render_cfg=rcfg, masks=masks, bbox=bbox)
    d_masks = t.from_numpy(np.stack([m.bits for m in masks]).astype(np.uint8)).to(cuda_device)
    b, tb = reconstruct_channel(images, cams, geom, hull, cfg, render_cfg=rcfg, masks=d_masks, bbox=bbox)
    assert np.array_equal(a.values, b.values)
    assert ta.rmse == tb.rmse


@pytest.mark.parametrize("shape", [(1, 1, 1), (5, 7, 3), (40, 33, 29)])
def test_hull_keypoints_match_key_point_mask(cuda_device, shape):
    from paper_1809_06417_b200.volume import HullTags

    t = _lib.torch()
    rng = np.random.default_rng(sum(shape))
    tags = np.where(rng.random(shape) < 0.2, 7, rng.integers(0, 7, shape)).astype(np.uint32)
    hull = HullTags(tags, 3)
    geom = VoxelGrid(*shape, np.zeros(3), 0.1)
    inside = t.from_numpy(hull.inside_voxels().astype(np.uint8)).to(cuda_device)
    kp = t.empty(geom.lattice_shape, dtype=t.uint8, device=cuda_device)
    vals = t.empty(geom.lattice_shape, dtype=t.float32, device=cuda_device)
    _lib.call("fvr_hull_keypoints", inside.data_ptr(), _lib.grid_struct(geom), kp.data_ptr(), vals.data_ptr(),
              _lib.stream_ptr())
    want = hull.key_point_mask()
    assert np.array_equal(kp.cpu().numpy().astype(bool), want)
    assert np.array_equal(vals.cpu().numpy(), np.where(want, np.float32(0), np.float32(-1)))


def test_save_volume_device_matches_host_writer(cuda_device, tmp_path):
    """FVR1 written from a device lattice (transpose on the GPU, pinned
    staging) is byte-identical to the host writer."""
    from paper_1809_06417_b200 import formats as F

    t = _lib.torch()
    rng = np.random.default_rng(2)
    geom = VoxelGrid(6, 5, 7, np.array([0.1, -0.2, 0.3]), 0.03)
    vals = (rng.random((3,) + geom.lattice_shape) * 200).astype(np.float32)
    grids = [VoxelGrid(6, 5, 7, geom.origin, geom.edge, tag, vals[c]) for c, tag in enumerate(("red", "green", "blue"))]
    F.save_volume(tmp_path / "h.fvr", grids)
    F.save_volume_device(tmp_path / "d.fvr", t.from_numpy(vals).to(cuda_device), geom)
    assert (tmp_path / "h.fvr").read_bytes() == (tmp_path / "d.fvr").read_bytes()
    back = F.load_volume(tmp_path / "d.fvr")
    assert all(np.array_equal(b.values, vals[c]) for c, b in enumerate(back))
