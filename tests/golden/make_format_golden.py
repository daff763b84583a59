"""Reference-written files for the format parity tests (§8f rank 4).

Runs the reference package (from the same scratch copy as make_golden.py)
and writes one small file per format into tests/golden/formats/, plus the
arrays they were written from (formats.npz):

    python tests/golden/make_format_golden.py
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "formats")
sys.path.insert(0, HERE)
from make_golden import _import_reference  # noqa: E402


def main():
    _import_reference()
    from fvr.imgio import Image, write_fim, write_pbm, write_ppm
    from fvr.volume import HullTags, VoxelGrid, save_hull, save_volume

    os.makedirs(OUT, exist_ok=True)
    rng = np.random.default_rng(5)
    nx, ny, nz = 3, 4, 5
    origin = np.array([-0.1, 0.05, 0.2])
    edge = 0.0125
    vals = (rng.random((3, nx + 1, ny + 1, nz + 1)) * 255).astype(np.float32)
    vals[:, 0, 0, :] = -1.0
    grids = [VoxelGrid(nx, ny, nz, origin, edge, t, vals[c]) for c, t in enumerate(("red", "green", "blue"))]
    save_volume(os.path.join(OUT, "rgb.fvr"), grids)
    save_volume(os.path.join(OUT, "temp.fvr"), [VoxelGrid(nx, ny, nz, origin, edge, "temperature", vals[1])])
    tags = rng.integers(0, 8, (nx, ny, nz)).astype(np.uint32)
    save_hull(os.path.join(OUT, "hull.fvh"), HullTags(tags, 3), grids[0])
    rgb = (rng.random((7, 9, 3)) * 300 - 20).clip(0, None).astype(np.float32)
    rgb[0, 0] = [254.5, 0.49, 255.0]
    gray = rgb[:, :, 1:2].copy()
    write_fim(os.path.join(OUT, "rgb.fim"), Image(9, 7, 3, rgb))
    write_fim(os.path.join(OUT, "gray.fim"), Image(9, 7, 1, gray))
    write_ppm(os.path.join(OUT, "rgb.ppm"), Image(9, 7, 3, rgb))
    write_ppm(os.path.join(OUT, "gray.pgm"), Image(9, 7, 1, gray))
    bits = rng.random((6, 11)) < 0.4
    write_pbm(os.path.join(OUT, "mask.pbm"), bits)
    np.savez_compressed(os.path.join(OUT, "formats.npz"), vals=vals, origin=origin, edge=edge, tags=tags, rgb=rgb,
                        gray=gray, bits=bits, dims=np.array([nx, ny, nz]))
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
