"""File formats (§8f rank 4) against files the reference itself wrote
(tests/golden/make_format_golden.py): readers recover the arrays exactly,
writers reproduce the reference's bytes, errors match (FormatError)."""

import os

import numpy as np
import pytest

from paper_1809_06417_b200 import FormatError, HullTags, Image, VoxelGrid
from paper_1809_06417_b200 import formats as F

GOLD = os.path.join(os.path.dirname(__file__), "golden", "formats")


@pytest.fixture(scope="module")
def ref():
    return np.load(os.path.join(GOLD, "formats.npz"))


def _grids(ref, tags=("red", "green", "blue")):
    nx, ny, nz = (int(x) for x in ref["dims"])
    return [VoxelGrid(nx, ny, nz, ref["origin"], float(ref["edge"]), t, ref["vals"][c]) for c, t in enumerate(tags)]


def _bytes(name):
    with open(os.path.join(GOLD, name), "rb") as f:
        return f.read()


def test_volume_read_write_byte_exact(ref, tmp_path):
    got = F.load_volume(os.path.join(GOLD, "rgb.fvr"))
    assert [g.channel_tag for g in got] == ["red", "green", "blue"]
    for c, g in enumerate(got):
        assert np.array_equal(g.values, ref["vals"][c])
        assert np.array_equal(g.origin, ref["origin"]) and g.edge == float(ref["edge"])
    F.save_volume(tmp_path / "rgb.fvr", _grids(ref))
    assert (tmp_path / "rgb.fvr").read_bytes() == _bytes("rgb.fvr")
    one = F.load_volume(os.path.join(GOLD, "temp.fvr"))
    assert len(one) == 1 and one[0].channel_tag == "temperature"
    assert np.array_equal(one[0].values, ref["vals"][1])


def test_hull_read_write_byte_exact(ref, tmp_path):
    hull, geom = F.load_hull(os.path.join(GOLD, "hull.fvh"))
    assert hull.n_views == 3 and np.array_equal(hull.tags, ref["tags"])
    assert geom.counts == tuple(int(x) for x in ref["dims"])
    F.save_hull(tmp_path / "h.fvh", HullTags(ref["tags"], 3), _grids(ref)[0])
    assert (tmp_path / "h.fvh").read_bytes() == _bytes("hull.fvh")


def test_images_byte_exact(ref, tmp_path):
    rgb, gray = ref["rgb"], ref["gray"]
    assert np.array_equal(F.read_fim(os.path.join(GOLD, "rgb.fim")).data, rgb)
    assert np.array_equal(F.load_image(os.path.join(GOLD, "gray.fim")).data, gray)
    F.write_fim(tmp_path / "a.fim", Image(9, 7, 3, rgb))
    assert (tmp_path / "a.fim").read_bytes() == _bytes("rgb.fim")
    F.write_ppm(tmp_path / "a.ppm", Image(9, 7, 3, rgb))
    F.write_ppm(tmp_path / "a.pgm", Image(9, 7, 1, gray))
    assert (tmp_path / "a.ppm").read_bytes() == _bytes("rgb.ppm")
    assert (tmp_path / "a.pgm").read_bytes() == _bytes("gray.pgm")
    back = F.load_image(os.path.join(GOLD, "rgb.ppm"))
    assert np.array_equal(back.data, F.quantize_u8(rgb).astype(np.float32))
    assert F.quantize_u8(np.array([254.5, 0.49, -3.0, 300.0])).tolist() == [255, 0, 0, 255]
    F.write_pbm(tmp_path / "m.pbm", ref["bits"])
    assert (tmp_path / "m.pbm").read_bytes() == _bytes("mask.pbm")
    assert np.array_equal(F.read_pbm(os.path.join(GOLD, "mask.pbm")), ref["bits"])


def test_format_errors(ref, tmp_path):
    p = tmp_path / "bad.fvr"
    p.write_bytes(b"FVR2" + _bytes("rgb.fvr")[4:])
    with pytest.raises(FormatError, match="bad magic"):
        F.load_volume(p)
    p.write_bytes(_bytes("rgb.fvr")[:-8])
    with pytest.raises(FormatError, match="truncated channel 2"):
        F.load_volume(p)
    p.write_bytes(_bytes("rgb.fvr")[:20])
    with pytest.raises(FormatError, match="truncated header"):
        F.load_volume(p)
    with pytest.raises(FormatError, match="3 channels but 1 tags"):
        F.load_volume(os.path.join(GOLD, "rgb.fvr"), tags=("x",))
    q = tmp_path / "bad.fim"
    q.write_bytes(_bytes("rgb.fim")[:4] + b"\x02\x00\x00\x00" + _bytes("rgb.fim")[8:])
    with pytest.raises(FormatError, match="unsupported version 2"):
        F.read_fim(q)
    r = tmp_path / "bad.ppm"
    r.write_bytes(b"P6\n2 2\n65535\n" + bytes(24))
    with pytest.raises(FormatError, match="only 8-bit"):
        F.read_ppm(r)
    with pytest.raises(ValueError):
        F.save_volume(tmp_path / "x.fvr", [])
