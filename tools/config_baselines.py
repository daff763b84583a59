"""BASELINE configs 3, 4 and 5 on one B200 next to the reference's CPU path
timed on the same box's host cores (profiles/r2_configs.jsonl).

  python tools/config_baselines.py 3|4|sweep [out.jsonl]

Configs 3 / 4: the device loop (ChannelLoop, render plan + adjust plan) timed
with CUDA events over 10 iterations after 3 warm-up ones, and the unmodified
reference (baseline/_ref, numba on all host threads) running one iteration
of the same workload through its public API: fvr.render.render_pixels of
two views' bbox pixels (scaled to all views) plus one fvr.reconstruct.adjust_pass
over every view (config 4: the reference allocates 16 partial lattices of
513^3 f64 = 17 GB for it).  Both use the same device-rendered inputs
(workloads.device_scene), handed to the reference as its own types.

Config 5 (render-only sweep): render_view of RGB grids on the device vs the
reference's render_pixels on a bounded sample of 2048 pixels of the first
view, scaled to the sweep point's full frames.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402


def ref_objects(ref, sc):
    R = ref["reconstruct"]
    geo = sys.modules["fvr.geometry"]
    vol = ref["volume"]
    pre = ref["preprocess"]
    cams = [geo.Camera(fx=c.fx, fy=c.fy, cx=c.cx, cy=c.cy, rotation=c.rotation, translation=c.translation,
                       width=c.width, height=c.height) for c in sc["cams"]]
    g = sc["geom"]
    geom = vol.VoxelGrid(g.nx, g.ny, g.nz, g.origin, g.edge)
    hull = vol.HullTags(sc["hull"].tags, len(cams))
    masks = [pre.FlameMask(m.width, m.height, m.bits) for m in sc["masks"]]
    b = sc["bbox"]
    bbox = pre.Rect(b.u0, b.v0, b.u1, b.v1)
    rcfg = ref["render"].RenderConfig(tau=sc["tau"], scattering_enabled=True, sigma_s=workloads.SIGMA_S,
                                      scatter_dirs=workloads.SCAT_DIRS)
    cfg = R.ReconstructionConfig(alpha_l=0.006, alpha_d=1.0, tau=sc["tau"], max_iters=1, converge_eps=1e-12,
                                 deterministic_mode=True)
    return cams, geom, hull, masks, bbox, rcfg, cfg


def cpu_iteration(sc):
    ref = workloads.import_reference()
    ref["kernels"].set_threads(os.cpu_count() or 1)
    cams, geom, hull, masks, bbox, rcfg, cfg = ref_objects(ref, sc)
    R = ref["reconstruct"]
    grid = R._init_grid(geom, hull, "green")
    uu, vv = np.meshgrid(np.arange(bbox.u0, bbox.u1 + 1) + 0.5, np.arange(bbox.v0, bbox.v1 + 1) + 0.5, indexing="xy")
    us, vs = uu.ravel(), vv.ravel()
    ref["render"].render_pixels(cams[0], [grid], rcfg, us[:64], vs[:64])  # JIT
    t0 = time.perf_counter()
    for v in (0, 1):
        ref["render"].render_pixels(cams[v], [grid], rcfg, us, vs)
    t_render = (time.perf_counter() - t0) / 2 * len(cams)
    src = [im.data[bbox.slices][:, :, 0].astype(np.float64) for im in sc["images"]]
    residuals = []
    for c, s in zip(cams, src):
        f = np.zeros((c.height, c.width))
        f[bbox.slices] = s  # residual of the initial (zero) grid: the image itself
        residuals.append(f)
    t0 = time.perf_counter()
    R.adjust_pass(grid, hull, cams, residuals, masks, cfg, np.random.default_rng(0), bbox)
    t_adjust = time.perf_counter() - t0
    return {"s_per_iter": t_render + t_adjust, "render_s": t_render, "adjust_s": t_adjust, "cores": os.cpu_count(),
            "kind": "reference",
            "sample": "render_pixels of 2 views' bbox pixels scaled to all views + one adjust_pass over all views"}


def gpu_loop(sc, iters=10):
    from paper_1809_06417_b200 import ReconstructionConfig
    from paper_1809_06417_b200.engine import ChannelLoop
    from paper_1809_06417_b200.reconstruct import _init_grid, _loop_config

    cfg = ReconstructionConfig(alpha_l=0.006, alpha_d=1.0, tau=sc["tau"], max_iters=iters + 3, converge_eps=1e-12,
                               deterministic_mode=True)
    grid0 = _init_grid(sc["geom"], sc["hull"], "green")
    src = [im.data[sc["bbox"].slices][:, :, 0] for im in sc["images"]]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    loop = ChannelLoop(sc["cams"], grid0, grid0.values, src, sc["masks"], sc["bbox"], sc["hull"].inside_voxels(),
                       sc["hull"].key_point_mask(), sc["rcfg"], _loop_config(cfg, grid0), cfg.max_iters,
                       background=0.0, use_graph=False)
    torch.cuda.synchronize()
    setup = time.perf_counter() - t0
    for _ in range(3):
        loop.launch_iteration()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        loop.launch_iteration()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    return {"ms_per_iter": ms, "iters_per_s": 1e3 / ms, "setup_s": setup, "hull_kp": loop.n_kp,
            "flame_rays": loop.n_rays, "render_plan_entries": loop.rplan_nnz, "adjust_plan_nnz": loop.plan_nnz,
            "render_path": "render plan" if loop.rplan else "marching kernel",
            "adjust_path": "gather plan" if loop.plan else "scatter"}


def config(cfg_no, out):
    n, views, res = workloads.CONFIGS[cfg_no]
    t0 = time.perf_counter()
    sc = workloads.device_scene(n, views, res)
    rec = {"config": cfg_no, "workload": workloads.workload_name(n, views, res), "scene_s": time.perf_counter() - t0}
    rec["gpu"] = gpu_loop(sc)
    if cfg_no == 3:
        from paper_1809_06417_b200 import build_color_temp_map, reconstruct_temperature

        cmap = build_color_temp_map()
        cfg = __import__("tests.fullsize_common", fromlist=["loop_cfg"]).loop_cfg(sc, 10)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = reconstruct_temperature(sc["rgb"], sc["cams"], cmap, sc["geom"], cfg, render_cfg=sc["rcfg"])
        rec["gpu"]["reconstruct_temperature_10_iters_s"] = time.perf_counter() - t0
        rec["gpu"]["temperature_clamped"] = [res.n_clamped_low, res.n_clamped_high]
    rec["cpu"] = cpu_iteration(sc)
    rec["gpu_over_cpu"] = rec["cpu"]["s_per_iter"] / (rec["gpu"]["ms_per_iter"] * 1e-3)
    print(json.dumps(rec), flush=True)
    with open(out, "a") as f:
        f.write(json.dumps(rec) + "\n")


def sweep(out):
    from paper_1809_06417_b200 import RenderConfig, _lib
    from paper_1809_06417_b200.radiometry import PhaseConfig
    from paper_1809_06417_b200.render import _RenderInputs, launch_render_views, prepare_render_inputs

    ref = workloads.import_reference()
    ref["kernels"].set_threads(os.cpu_count() or 1)
    geo = sys.modules["fvr.geometry"]
    vol = ref["volume"]
    peak = json.load(open(os.path.join(workloads.ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    for n in (64, 128, 256, 512):
        res = 512 if n <= 128 else 1024
        sc = workloads.device_scene(n, 32, res, scattering=False)
        rgrids = [vol.VoxelGrid(g.nx, g.ny, g.nz, g.origin, g.edge, g.channel_tag, g.values) for g in sc["truth"]]
        c0 = sc["cams"][0]
        rcam = geo.Camera(fx=c0.fx, fy=c0.fy, cx=c0.cx, cy=c0.cy, rotation=c0.rotation, translation=c0.translation,
                          width=c0.width, height=c0.height)
        rng = np.random.default_rng(0)
        us = rng.integers(0, res, 2048) + 0.5
        vs = rng.integers(0, res, 2048) + 0.5
        for views in (4, 8, 16, 32):
            cams = sc["cams"][:views]
            for scattering in (False, True):
                cfg = RenderConfig(tau=workloads.tau_n(n), scattering_enabled=scattering,
                                   sigma_s=0.1 if scattering else 0.0)
                inp = _RenderInputs(sc["truth"], cfg, PhaseConfig(0.0))
                prepare_render_inputs(inp)
                cams_t = _lib.cameras_tensor(cams, inp.dev)
                out_t = torch.empty((views, res, res, 3), dtype=torch.float32, device=inp.dev)
                launch_render_views(inp, cams_t, views, res, res, out_t)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(3):
                    launch_render_views(inp, cams_t, views, res, res, out_t)
                e1.record()
                torch.cuda.synchronize()
                gpu_s = e0.elapsed_time(e1) / 3e3
                rec = {"config": 5, "n": n, "views": views, "res": res, "scattering": scattering, "gpu_ms": gpu_s * 1e3,
                       "gpu_views_per_s": views / gpu_s}
                if views == 4:  # the CPU sample once per (n, scattering): 2048 pixels of one view
                    rc = ref["render"].RenderConfig(tau=workloads.tau_n(n), scattering_enabled=scattering,
                                                    sigma_s=0.1 if scattering else 0.0)
                    ref["render"].render_pixels(rcam, rgrids, rc, us[:8], vs[:8])
                    t0 = time.perf_counter()
                    ref["render"].render_pixels(rcam, rgrids, rc, us, vs)
                    cpu_px = (time.perf_counter() - t0) / us.size
                    rec["cpu_views_per_s"] = 1.0 / (cpu_px * res * res)
                    rec["cpu_sample"] = "reference render_pixels of 2048 random pixels of view 0, RGB, scaled to a frame"
                    rec["cpu_cores"] = os.cpu_count()
                print(json.dumps(rec), flush=True)
                with open(out, "a") as f:
                    f.write(json.dumps(rec) + "\n")
        del sc
        torch.cuda.empty_cache()
    del peak


if __name__ == "__main__":
    torch.cuda.set_device(0)
    what = sys.argv[1]
    out = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/r2_configs.jsonl"
    if what == "sweep":
        sweep(out)
    else:
        config(int(what), out)
