"""File formats of the reference package (§8f rank 4), byte-compatible:

* FVR1 volumes  -- volume.py:335-398 (save_volume / load_volume)
* FVH1 hull tags -- volume.py:401-440 (save_hull / load_hull)
* FIM1 float images -- imgio.py:140-178 (write_fim / read_fim / load_image)
* binary PNM (P5/P6 8-bit, P4 bitmaps) -- imgio.py:56-137

All multi-byte fields are little-endian.  Volumes and hulls are stored
x-fastest (Fortran order) while the in-memory lattice is C order (z
fastest), so writers transpose; ``save_volume_device`` does that transpose on
the GPU and streams the planes through page-locked memory, which keeps the
host out of the way when snapshots are written during a reconstruction.
"""

from __future__ import annotations

import struct

import numpy as np

from .errors import FormatError
from .imgio import Image

MAGIC_VOLUME = b"FVR1"
MAGIC_HULL = b"FVH1"
MAGIC_IMAGE = b"FIM1"

# magic, version, count (channels / views), nx, ny, nz, origin xyz, edge
_GRID_HEAD = struct.Struct("<4sIIIII3dd")
# magic, version, channels, width, height
_IMAGE_HEAD = struct.Struct("<4sIIII")


def _read_head(f, spec: struct.Struct, magic: bytes, path):
    raw = f.read(spec.size)
    if len(raw) < spec.size:
        raise FormatError(f"{path}: truncated header")
    fields = spec.unpack(raw)
    if fields[0] != magic:
        raise FormatError(f"{path}: bad magic {fields[0]!r}")
    if fields[1] != 1:
        raise FormatError(f"{path}: unsupported version {fields[1]}")
    return fields[2:]


def _read_exact(f, n: int, path, what: str) -> bytes:
    buf = f.read(n)
    if len(buf) < n:
        raise FormatError(f"{path}: truncated {what}")
    return buf


# --- volumes ------------------------------------------------------------------


def save_volume(path, grids) -> None:
    """C planes of f32 key-point values, x-fastest, after the FVR1 header."""
    grids = list(grids)
    if not grids:
        raise ValueError("no grids to save")
    g0 = grids[0]
    if any(not g0.same_geometry(g) for g in grids[1:]):
        raise ValueError("all channels must share geometry")
    with open(path, "wb") as f:
        f.write(_GRID_HEAD.pack(MAGIC_VOLUME, 1, len(grids), g0.nx, g0.ny, g0.nz, *map(float, g0.origin),
                                float(g0.edge)))
        for g in grids:
            f.write(np.asarray(g.values, dtype="<f4").transpose(2, 1, 0).tobytes())


def save_volume_device(path, values, grid_geom) -> None:
    """FVR1 straight from a device lattice ``values`` ((C,) + lattice f32
    tensor): the x-fastest transpose runs on the GPU and each plane comes
    back through one page-locked buffer."""
    from . import _lib

    t = _lib.torch()
    vals = values if values.dim() == 4 else values.unsqueeze(0)
    shape = (grid_geom.nx + 1, grid_geom.ny + 1, grid_geom.nz + 1)
    if tuple(vals.shape[1:]) != shape:
        raise ValueError(f"lattice shape {tuple(vals.shape[1:])} != grid {shape}")
    staging = t.empty(shape[::-1], dtype=t.float32, pin_memory=True)
    with open(path, "wb") as f:
        f.write(_GRID_HEAD.pack(MAGIC_VOLUME, 1, vals.shape[0], grid_geom.nx, grid_geom.ny, grid_geom.nz,
                                *map(float, grid_geom.origin), float(grid_geom.edge)))
        for c in range(vals.shape[0]):
            staging.copy_(vals[c].permute(2, 1, 0))
            f.write(staging.numpy().tobytes())


def load_volume(path, tags: tuple[str, ...] | None = None):
    from .volume import VoxelGrid

    with open(path, "rb") as f:
        nch, nx, ny, nz, ox, oy, oz, edge = _read_head(f, _GRID_HEAD, MAGIC_VOLUME, path)
        if tags is None:
            tags = ("red", "green", "blue") if nch == 3 else ("temperature",) * nch
        if len(tags) != nch:
            raise FormatError(f"{path}: {nch} channels but {len(tags)} tags given")
        n = (nx + 1) * (ny + 1) * (nz + 1)
        out = []
        for c in range(nch):
            plane = np.frombuffer(_read_exact(f, 4 * n, path, f"channel {c}"), dtype="<f4")
            lattice = plane.reshape(nz + 1, ny + 1, nx + 1).transpose(2, 1, 0)
            out.append(VoxelGrid(nx, ny, nz, np.array([ox, oy, oz]), edge, tags[c], lattice))
    return out


def save_hull(path, hull, grid_geom) -> None:
    with open(path, "wb") as f:
        f.write(_GRID_HEAD.pack(MAGIC_HULL, 1, hull.n_views, grid_geom.nx, grid_geom.ny, grid_geom.nz,
                                *map(float, grid_geom.origin), float(grid_geom.edge)))
        f.write(np.asarray(hull.tags, dtype="<u4").transpose(2, 1, 0).tobytes())


def load_hull(path):
    """(HullTags, empty VoxelGrid carrying the hull's geometry)."""
    from .volume import HullTags, VoxelGrid

    with open(path, "rb") as f:
        n_views, nx, ny, nz, ox, oy, oz, edge = _read_head(f, _GRID_HEAD, MAGIC_HULL, path)
        raw = _read_exact(f, 4 * nx * ny * nz, path, "tag data")
    tags = np.frombuffer(raw, dtype="<u4").reshape(nz, ny, nx).transpose(2, 1, 0)
    return HullTags(np.ascontiguousarray(tags), n_views), VoxelGrid(nx, ny, nz, np.array([ox, oy, oz]), edge)


# --- images -------------------------------------------------------------------


def write_fim(path, img: Image) -> None:
    """Lossless f32 planes (one per channel, row-major) after the FIM1 header."""
    with open(path, "wb") as f:
        f.write(_IMAGE_HEAD.pack(MAGIC_IMAGE, 1, img.channels, img.width, img.height))
        f.write(np.asarray(img.data, dtype="<f4").transpose(2, 0, 1).tobytes())


def read_fim(path) -> Image:
    with open(path, "rb") as f:
        channels, width, height = _read_head(f, _IMAGE_HEAD, MAGIC_IMAGE, path)
        planes = [np.frombuffer(_read_exact(f, 4 * width * height, path, f"channel {c}"), dtype="<f4")
                  for c in range(channels)]
    return Image(width, height, channels, np.stack(planes, axis=-1).reshape(height, width, channels))


def quantize_u8(data: np.ndarray) -> np.ndarray:
    """Clamp to [0, 255] and round half up."""
    return np.floor(np.clip(data, 0.0, 255.0) + 0.5).astype(np.uint8)


def write_ppm(path, img: Image) -> None:
    """P6 for RGB, P5 for grayscale, 8-bit."""
    px = quantize_u8(img.data)
    header = b"%s\n%d %d\n255\n" % (b"P6" if img.channels == 3 else b"P5", img.width, img.height)
    with open(path, "wb") as f:
        f.write(header + (px if img.channels == 3 else px[:, :, 0]).tobytes())


def _pnm_tokens(f, path, count: int) -> list[bytes]:
    """The first ``count`` whitespace-separated header tokens (# comments skipped)."""
    out, tok = [], b""
    while len(out) < count:
        ch = f.read(1)
        if not ch:
            raise FormatError(f"{path}: truncated header")
        if ch == b"#" and not tok:
            while ch not in (b"\n", b""):
                ch = f.read(1)
        elif ch.isspace():
            if tok:
                out.append(tok)
                tok = b""
        else:
            tok += ch
    return out


def read_ppm(path) -> Image:
    with open(path, "rb") as f:
        magic, w, h, maxval = _pnm_tokens(f, path, 4)
        if magic not in (b"P5", b"P6"):
            raise FormatError(f"{path}: unsupported magic {magic!r}")
        if int(maxval) != 255:
            raise FormatError(f"{path}: only 8-bit images supported, maxval={int(maxval)}")
        w, h = int(w), int(h)
        ch = 3 if magic == b"P6" else 1
        raw = _read_exact(f, w * h * ch, path, "pixel data")
    return Image(w, h, ch, np.frombuffer(raw, dtype=np.uint8).reshape(h, w, ch).astype(np.float32))


def write_pbm(path, bits) -> None:
    """P4 bitmap, rows padded to whole bytes; set bits are black."""
    bits = np.asarray(bits, dtype=bool)
    with open(path, "wb") as f:
        f.write(b"P4\n%d %d\n" % (bits.shape[1], bits.shape[0]) + np.packbits(bits, axis=1).tobytes())


def read_pbm(path) -> np.ndarray:
    with open(path, "rb") as f:
        magic, w, h = _pnm_tokens(f, path, 3)
        if magic != b"P4":
            raise FormatError(f"{path}: not a P4 PBM")
        w, h = int(w), int(h)
        stride = (w + 7) // 8
        raw = _read_exact(f, stride * h, path, "bitmap")
    return np.unpackbits(np.frombuffer(raw, dtype=np.uint8).reshape(h, stride), axis=1)[:, :w].astype(bool)


def load_image(path) -> Image:
    """FIM1 or binary PPM/PGM, by content."""
    with open(path, "rb") as f:
        head = f.read(4)
    return read_fim(path) if head == MAGIC_IMAGE else read_ppm(path)
