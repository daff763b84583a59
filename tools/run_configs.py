"""Timing of the other BASELINE configs on one GPU (diagnostic; results go to
profiles/).  config 3: 256^3 x 16 views 1024^2, full RTE + temperature;
config 4: 512^3 x 32 views 1024^2, full RTE (1 GPU here; the 8-GPU run
shards the views); config 5: render-only sweep.

  python tools/run_configs.py 3 [iters]      python tools/run_configs.py sweep
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch


def tau_n(n):
    return 1.0 - 0.95 ** (64.0 / n) if n >= 128 else 0.05


def scene(n, views, res, scattering=True):
    from paper_1809_06417_b200 import RenderConfig, VoxelGrid, compute_visual_hull, render_view
    from paper_1809_06417_b200.preprocess import bounding_box, threshold_mask
    from paper_1809_06417_b200.synth import synth_cameras, synth_volume

    t0 = time.perf_counter()
    vols = synth_volume((n, n, n), seed=0, kind="flame")
    t_synth = time.perf_counter() - t0
    truth = [vols[t] for t in ("red", "green", "blue")]
    cams = synth_cameras(views, radius=0.38, fov=60.0, elevation_jitter_deg=5.0, width=res, height=res, seed=0)
    rcfg = RenderConfig(tau=tau_n(n), scattering_enabled=scattering, sigma_s=0.1 if scattering else 0.0,
                        scatter_dirs=32)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    imgs = [render_view(c, truth, None, rcfg) for c in cams]
    torch.cuda.synchronize()
    t_render = time.perf_counter() - t0
    masked = [threshold_mask(im) for im in imgs]
    masks = [m for m, _ in masked]
    bbox = bounding_box(masks, 4)
    geom = VoxelGrid(n, n, n, truth[0].origin, truth[0].edge)
    t0 = time.perf_counter()
    hull = compute_visual_hull(geom, [m.bits for m in masks], cams)
    t_hull = time.perf_counter() - t0
    return dict(truth=truth, vols=vols, cams=cams, rcfg=rcfg, imgs=imgs, masks=masks,
                blanked=[im for _, im in masked], bbox=bbox, geom=geom, hull=hull,
                t_synth=t_synth, t_render_inputs=t_render, t_hull=t_hull)


def loop_config(n, views, res, iters, temperature):
    from paper_1809_06417_b200 import ReconstructionConfig, build_color_temp_map
    from paper_1809_06417_b200.engine import ChannelLoop
    from paper_1809_06417_b200.reconstruct import _init_grid, _loop_config, green_to_temperature

    sc = scene(n, views, res)
    cfg = ReconstructionConfig(alpha_l=0.006, alpha_d=1.0, tau=tau_n(n), max_iters=iters + 3, converge_eps=1e-12,
                               deterministic_mode=True)
    grid0 = _init_grid(sc["geom"], sc["hull"], "green")
    src = [im.data[sc["bbox"].slices][:, :, 1] for im in sc["blanked"]]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    loop = ChannelLoop(sc["cams"], grid0, grid0.values, src, sc["masks"], sc["bbox"], sc["hull"].inside_voxels(),
                       sc["hull"].key_point_mask(), sc["rcfg"], _loop_config(cfg, grid0), cfg.max_iters,
                       background=0.0, use_graph=False)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0
    stream = torch.cuda.current_stream().cuda_stream
    for _ in range(3):
        loop.launch_iteration()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        loop.launch_iteration()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    st = loop.read_state()
    out = dict(config=f"{n}^3 x {views} views {res}^2, full RTE", iters=iters, ms_per_iter=ms, iters_per_s=1e3 / ms,
               setup_s=t_setup, plan_nnz=loop.plan_nnz, hull_kp=loop.n_kp, flame_rays=loop.n_rays,
               bbox=[sc["bbox"].u0, sc["bbox"].v0, sc["bbox"].u1, sc["bbox"].v1],
               rmse_first=float(loop.trace[0, 0].item()), rmse_last=float(loop.trace[0, st["it"] - 1].item()),
               synth_s=sc["t_synth"], render_inputs_s=sc["t_render_inputs"], hull_s=sc["t_hull"],
               max_mem_gb=torch.cuda.max_memory_allocated() / 1e9)
    if temperature:
        cmap = build_color_temp_map()
        from paper_1809_06417_b200.volume import VoxelGrid

        g = VoxelGrid(n, n, n, sc["geom"].origin, sc["geom"].edge, "green", loop.host_values())
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        tg, lo, hi = green_to_temperature(g, cmap, sc["hull"].key_point_mask())
        torch.cuda.synchronize()
        out.update(temperature_s=time.perf_counter() - t0, n_clamped_low=lo, n_clamped_high=hi,
                   temp_range=[float(tg.values[tg.values > 0].min()), float(tg.values.max())])
    print(json.dumps(out))


def count_samples(cams, geom) -> int:
    """Render samples of full frames (slab clip + floor count, numpy fp64)."""
    from paper_1809_06417_b200.geometry import pixel_rays

    lo = geom.origin
    hi = lo + np.array([geom.nx, geom.ny, geom.nz]) * geom.edge
    total = 0
    for cam in cams:
        uu, vv = np.meshgrid(np.arange(cam.width) + 0.5, np.arange(cam.height) + 0.5, indexing="xy")
        o, d = pixel_rays(cam, uu.ravel(), vv.ravel())
        with np.errstate(divide="ignore", invalid="ignore"):
            t0 = (lo - o) / d
            t1 = (hi - o) / d
        tmin = np.max(np.where(d == 0, -1e300, np.minimum(t0, t1)), axis=1)
        tmax = np.min(np.where(d == 0, 1e300, np.maximum(t0, t1)), axis=1)
        te = np.maximum(tmin, 0.0)
        total += int(np.where(tmax > te, np.floor((tmax - te) / geom.edge + 1e-9), 0).sum())
    return total


def sweep():
    """Config 5: forward RTE of RGB grids, inputs resident, one batched launch
    per (n, V); device time from CUDA events."""
    from paper_1809_06417_b200 import RenderConfig, _lib
    from paper_1809_06417_b200.render import _RenderInputs, launch_render_views, prepare_render_inputs
    from paper_1809_06417_b200.radiometry import PhaseConfig

    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json")))["hbm_gbs"]
    for n in (64, 128, 256, 512):
        res = 512 if n <= 128 else 1024
        sc = scene(n, 32, res, scattering=False)
        for views in (4, 8, 16, 32):
            cams = sc["cams"][:views]
            samples = count_samples(cams, sc["geom"])
            for scattering in (False, True):
                cfg = RenderConfig(tau=tau_n(n), scattering_enabled=scattering, sigma_s=0.1 if scattering else 0.0)
                inp = _RenderInputs(sc["truth"], cfg, PhaseConfig(0.0))
                prepare_render_inputs(inp)
                cams_t = _lib.cameras_tensor(cams, inp.dev)
                out = torch.empty((views, res, res, 3), dtype=torch.float32, device=inp.dev)
                launch_render_views(inp, cams_t, views, res, res, out)  # warm
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                reps = 3
                e0.record()
                for _ in range(reps):
                    launch_render_views(inp, cams_t, views, res, res, out)
                e1.record()
                torch.cuda.synchronize()
                sec = e0.elapsed_time(e1) / 1e3 / reps
                bytes_alg = (108 if scattering else 32) * 3 * samples
                row = dict(n=n, views=views, res=res, scattering=scattering, ms=sec * 1e3, samples=samples,
                           gsamples_per_s=samples / sec / 1e9, alg_gbs=bytes_alg / sec / 1e9,
                           alg_frac=bytes_alg / sec / 1e9 / peak)
                print(json.dumps(row), flush=True)
        del sc
        torch.cuda.empty_cache()


if __name__ == "__main__":
    torch.cuda.set_device(0)
    what = sys.argv[1]
    if what == "sweep":
        sweep()
    else:
        n, views, res = {"2": (128, 8, 512), "3": (256, 16, 1024), "4": (512, 32, 1024)}[what]
        loop_config(n, views, res, int(sys.argv[2]) if len(sys.argv) > 2 else 10, temperature=(what == "3"))
