"""The BASELINE.json workloads, shared by bench.py, the
full-size GPU parity tests and tools/.

Inputs follow the §8(d) recipe: ``synth_volume((n,)*3, seed=0,
kind="flame")``, ``synth_cameras(V, radius=0.38, fov=60,
elevation_jitter_deg=5, seed=0)`` at res x res, RGB views rendered with the
loop's own RenderConfig, masks from ``threshold_mask`` (> 30), the union
bbox dilated by 4 pixels, the visual hull, and tau_n = 1 - 0.95^(64/n).

``device_scene`` builds them with this package (the GPU arm and the parity
tests); ``reference_scene`` builds them with the unmodified reference
installed in ``baseline/_ref`` (the reference arm of bench.py), so that arm
never loads this package or its library.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(ROOT, "baseline", "_ref")

# config number -> (n voxels per axis, views, resolution); BASELINE.json configs[0..3]
CONFIGS = {1: (32, 4, 64), 2: (128, 8, 512), 3: (256, 16, 1024), 4: (512, 32, 1024)}
SIGMA_S = 0.1
SCAT_DIRS = 32
ALPHA_L = 0.006
L2_NOTE = ("no flush: inputs larger than L2 -- every step streams the render and adjust plans (0.75 GB at "
           "config 2) through the 126 MB L2")


def tau_n(n: int) -> float:
    """Constant physical opacity anchored at the validated 64^3 scene (§8d);
    config 1 keeps the reference default 0.05."""
    return 1.0 - 0.95 ** (64.0 / n) if n >= 128 else 0.05


def workload_name(n: int, views: int, res: int, scattering: bool = True) -> str:
    cfg = {v: k for k, v in CONFIGS.items()}.get((n, views, res))
    rte = "full RTE (sigma_s 0.1, 32 dirs)" if scattering else "emission + extinction"
    head = f"config {cfg}: " if cfg else ""
    return f"{head}{n}^3 flame, {views} views {res}x{res}, {rte}, green channel"


def bench_config(n: int, views: int, res: int, bbox, world: int, scattering: bool = True) -> dict:
    """The ``config`` object of a bench line; both arms print exactly this."""
    return {"workload": workload_name(n, views, res, scattering), "n": n, "views": views, "res": res,
            "tau": tau_n(n), "sigma_s": SIGMA_S if scattering else 0.0, "scatter_dirs": SCAT_DIRS,
            "bbox": [int(b) for b in bbox], "parallelism": f"view-sharded x{world}" if world > 1 else "1 GPU",
            "l2": L2_NOTE}


def device_scene(n: int, views: int, res: int, scattering: bool = True) -> dict:
    """The workload's inputs, rendered and carved on the device."""
    from paper_1809_06417_b200 import RenderConfig, VoxelGrid, compute_visual_hull, render_view
    from paper_1809_06417_b200.preprocess import bounding_box, threshold_mask
    from paper_1809_06417_b200.synth import synth_cameras, synth_volume

    t0 = time.perf_counter()
    vols = synth_volume((n, n, n), seed=0, kind="flame")
    truth = [vols[t] for t in ("red", "green", "blue")]
    cams = synth_cameras(views, radius=0.38, fov=60.0, elevation_jitter_deg=5.0, width=res, height=res, seed=0)
    rcfg = RenderConfig(tau=tau_n(n), scattering_enabled=scattering, sigma_s=SIGMA_S if scattering else 0.0,
                        scatter_dirs=SCAT_DIRS)
    imgs = [render_view(c, truth, None, rcfg) for c in cams]
    masked = [threshold_mask(im) for im in imgs]
    masks = [m for m, _ in masked]
    blanked = [im for _, im in masked]
    bbox = bounding_box(masks, 4)
    geom = VoxelGrid(n, n, n, truth[0].origin, truth[0].edge)
    hull = compute_visual_hull(geom, [m.bits for m in masks], cams)
    return dict(n=n, views=views, res=res, tau=tau_n(n), truth=truth, temperature=vols["temperature"], cams=cams,
                rcfg=rcfg, rgb=imgs, blanked=blanked, images=[im.channel(1) for im in blanked], masks=masks,
                bbox=bbox, geom=geom, hull=hull, setup_s=time.perf_counter() - t0)


def reference_available() -> bool:
    return os.path.isdir(os.path.join(REF_DIR, "fvr"))


def import_reference():
    """The unmodified reference package from baseline/_ref (installed with
    pip --target; DESIGN.md §6 records the install)."""
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import fvr  # noqa: F401
    from fvr import _kernels, preprocess, reconstruct, render, synth, volume

    return dict(kernels=_kernels, preprocess=preprocess, reconstruct=reconstruct, render=render, synth=synth,
                volume=volume)


def reference_scene(n: int, views: int, res: int, scattering: bool = True) -> dict:
    """The same workload built by the reference itself on the host cores:
    fvr.synth, fvr.render.render_view, fvr.preprocess, compute_visual_hull."""
    ref = import_reference()
    ref["kernels"].set_threads(os.cpu_count() or 1)
    t0 = time.perf_counter()
    vols = ref["synth"].synth_volume((n, n, n), seed=0, kind="flame")
    truth = [vols[t] for t in ("red", "green", "blue")]
    cams = ref["synth"].synth_cameras(views, radius=0.38, fov=60.0, elevation_jitter_deg=5.0, width=res,
                                      height=res, seed=0)
    rcfg = ref["render"].RenderConfig(tau=tau_n(n), scattering_enabled=scattering,
                                      sigma_s=SIGMA_S if scattering else 0.0, scatter_dirs=SCAT_DIRS)
    imgs = [ref["render"].render_view(c, truth, None, rcfg) for c in cams]
    masked = [ref["preprocess"].threshold_mask(im) for im in imgs]
    masks = [m for m, _ in masked]
    bbox = ref["preprocess"].bounding_box(masks, 4)
    geom = ref["volume"].VoxelGrid(n, n, n, truth[0].origin, truth[0].edge)
    hull = ref["volume"].compute_visual_hull(geom, [m.bits for m in masks], cams)
    images = [im.channel(1) for _, im in masked]
    return dict(ref=ref, n=n, views=views, res=res, tau=tau_n(n), cams=cams, rcfg=rcfg, images=images,
                masks=masks, bbox=bbox, geom=geom, hull=hull, setup_s=time.perf_counter() - t0)
