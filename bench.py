#!/usr/bin/env python
"""Benchmark of the reconstruction loop (BASELINE.json metric and configs[1]).

Workload (configs[1]): 128^3 synthetic flame (synth_volume seed 0), 8 views of
512x512 (synth_cameras radius 0.38, fov 60, jitter 5, seed 0), full RTE
(emission, extinction, single scattering sigma_s = 0.1 over 32 Fibonacci
directions), tau_n = 1 - 0.95^(64/n) = 0.02532, green channel, deterministic
G, alpha_l = 0.006, alpha_d = 1, converge_eps = 1e-12 so every iteration runs.
A step is one reconstruction iteration: render + residual + RMSE of every
bbox pixel of every view, back-projection of every flame ray, convergence
rule, clamped update.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Prints one JSON line (rank 0).  Multi-GPU runs are launched by torchrun:
views are sharded across ranks and one NCCL all-reduce per iteration sums
the corrections (engine.py); time is the max over ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_VOX = 128
N_VIEWS = 8
RES = 512
SIGMA_S = 0.1
SCAT_DIRS = 32
TAU = 1.0 - 0.95 ** (64.0 / N_VOX)
ALPHA_L = 0.006
# dram__bytes_read.sum + dram__bytes_write.sum of K-render from one `ncu --set full`
# capture: the render-plan SpMV (profiles/r1_ncu_final9_render_gather_raw.csv) and the marching
# kernel it replaced (profiles/r1_ncu_render_final_raw.csv)
TRAFFIC_BYTES_PER_LAUNCH = {"rplan_render_kernel<1>": 522_099_968, "loop_render_scat_kernel": 10_210_304}
TRAFFIC_SOURCE = {"rplan_render_kernel<1>": "profiles/r2final_ncu_det_raw.csv (round 2 final, ID 0)",
                  "loop_render_scat_kernel": "profiles/r1_ncu_render_final_raw.csv (round 1)"}
# a pure 32-byte-load read stream over 2 GiB on a B200 of this pool (best variant, median of 20 launches)
READ_STREAM_GBS = 7261.3
READ_STREAM_SOURCE = "profiles/r2_read_peak.json (tools/read_peak.cu)"
DTYPE = ("f32 values, 17-bit-mantissa operator weights (render and adjust plans), f64 geometry, "
         "32.32 fixed-point accumulation")
METRIC = "recon iters/sec at 128³×8 views 512²; Gsamples/s; % of HBM roofline"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# inputs
# ---------------------------------------------------------------------------


def make_scene():
    """Synthetic inputs of configs[1], rendered on the device (workloads.py)."""
    import workloads

    return workloads.device_scene(N_VOX, N_VIEWS, RES)


def work_counts(sc):
    """S_r (render samples), S_f (samples on flame rays), S_a (in-hull adjust
    samples), R_f, V*P, N_kp per iteration, counted exactly."""
    from paper_1809_06417_b200 import _kernels
    from paper_1809_06417_b200.geometry import pixel_rays

    geom, bbox = sc["geom"], sc["bbox"]
    lo = geom.origin
    hi = lo + np.array([geom.nx, geom.ny, geom.nz]) * geom.edge
    us = np.arange(bbox.u0, bbox.u1 + 1) + 0.5
    vs = np.arange(bbox.v0, bbox.v1 + 1) + 0.5
    uu, vv = np.meshgrid(us, vs, indexing="xy")

    def samples(o, d):
        with np.errstate(divide="ignore", invalid="ignore"):
            t0 = (lo[None, :] - o[None, :]) / d
            t1 = (hi[None, :] - o[None, :]) / d
        tmin = np.max(np.where(d == 0, -1e300, np.minimum(t0, t1)), axis=1)
        tmax = np.min(np.where(d == 0, 1e300, np.maximum(t0, t1)), axis=1)
        te = np.maximum(tmin, 0.0)
        n = np.floor((tmax - te) / geom.edge + 1e-9)
        return np.where(tmax > te, n, 0).astype(np.int64)

    inside = sc["hull"].inside_voxels().astype(np.uint8)
    s_r = s_f = s_a = r_f = 0
    for cam, mask in zip(sc["cams"], sc["masks"]):
        o, d = pixel_rays(cam, uu.ravel(), vv.ravel())
        s_r += int(samples(o, d).sum())
        rows, cols = np.nonzero(mask.bits[bbox.slices])
        fo, fd = pixel_rays(cam, cols + bbox.u0 + 0.5, rows + bbox.v0 + 0.5)
        s_f += int(samples(fo, fd).sum())
        counts = np.empty(rows.size, dtype=np.int64)
        _kernels.count_hull_samples(fo, fd, inside, geom.origin, geom.edge, counts)
        s_a += int(counts.sum())
        r_f += int(rows.size)
    vp = len(sc["cams"]) * bbox.area
    n_kp = (geom.nx + 1) * (geom.ny + 1) * (geom.nz + 1)
    return dict(S_r=s_r, S_f=s_f, S_a=s_a, R_f=r_f, VP=vp, N_kp=n_kp,
                hull_kp=int(sc["hull"].key_point_mask().sum()))


def live_samples(sc, occ) -> int:
    """Render samples whose 3x3x3 neighbourhood may be non-zero (distance map <= 1; the ones K-render
    evaluates; the rest add exactly 0 and are skipped), counted on the device
    with torch in fp64 from the same q = qb + k*d as the kernel."""
    import torch

    from paper_1809_06417_b200.geometry import pixel_rays

    geom, bbox = sc["geom"], sc["bbox"]
    dev = occ.device
    lo = torch.tensor(geom.origin, dtype=torch.float64, device=dev)
    n = torch.tensor([geom.nx, geom.ny, geom.nz], dtype=torch.float64, device=dev)
    hi = lo + n * geom.edge
    occ_flat = occ.reshape(-1)
    sx, sy = (geom.ny + 1) * (geom.nz + 1), geom.nz + 1
    us = np.arange(bbox.u0, bbox.u1 + 1) + 0.5
    vs = np.arange(bbox.v0, bbox.v1 + 1) + 0.5
    uu, vv = np.meshgrid(us, vs, indexing="xy")
    live = 0
    for cam in sc["cams"]:
        o_np, d_np = pixel_rays(cam, uu.ravel(), vv.ravel())
        o = torch.tensor(o_np, dtype=torch.float64, device=dev)
        for chunk in np.array_split(np.arange(d_np.shape[0]), 8):
            d = torch.tensor(d_np[chunk], dtype=torch.float64, device=dev)
            with np.errstate(all="ignore"):
                t0 = (lo - o) / d
                t1 = (hi - o) / d
            tmin = torch.where(d == 0, torch.full_like(d, -1e300), torch.minimum(t0, t1)).amax(1)
            tmax = torch.where(d == 0, torch.full_like(d, 1e300), torch.maximum(t0, t1)).amin(1)
            te = tmin.clamp(min=0.0)
            cnt = torch.where(tmax > te, torch.floor((tmax - te) / geom.edge + 1e-9), torch.zeros_like(te)).long()
            kmax = int(cnt.max().item()) if cnt.numel() else 0
            if kmax == 0:
                continue
            qb = ((o - lo)[None, :] + (te - 0.5 * geom.edge)[:, None] * d) / geom.edge
            k = torch.arange(1, kmax + 1, dtype=torch.float64, device=dev)
            q = qb[:, None, :] + k[None, :, None] * d[:, None, :]
            m = torch.round(q).long()
            m = torch.minimum(torch.clamp(m, min=0), n.long())
            idx = m[..., 0] * sx + m[..., 1] * sy + m[..., 2]
            valid = k[None, :] <= cnt[:, None]
            live += int(((occ_flat[idx.clamp(max=occ_flat.numel() - 1)] <= 1) & valid).sum().item())
    return live


def algorithmic_bytes(w, scattering=True):
    """B_iter = 32 S_r [+76 S_r with scattering] + 64 S_a +
    1 S_f + 8 V P + 4 R_f + 16 N_kp."""
    render = (108 if scattering else 32) * w["S_r"] + 8 * w["VP"]
    total = render + 64 * w["S_a"] + w["S_f"] + 4 * w["R_f"] + 16 * w["N_kp"]
    return render, total


# ---------------------------------------------------------------------------
# clocks
# ---------------------------------------------------------------------------


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def wait_first(self, timeout: float = 5.0) -> None:
        """Block until nvidia-smi delivered its first row (its start-up can
        outlast a short timed region)."""
        t_end = time.time() + timeout
        while self.proc is not None and not self.rows and time.time() < t_end:
            time.sleep(0.02)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        time.sleep(0.05)
        rows = self.rows
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None

        sm = [num(r[1]) for r in rows if num(r[1]) is not None]
        mx = [num(r[2]) for r in rows if num(r[2]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------


def run_gpu(args):
    import torch

    import ctypes

    import workloads
    from paper_1809_06417_b200 import ReconstructionConfig, _lib, reconstruct_channel
    from paper_1809_06417_b200.engine import ChannelLoop
    from paper_1809_06417_b200.reconstruct import _init_grid, _loop_config

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # FVR_BENCH_ONE_GPU=1 (tests only): every rank on cuda:0 over gloo, to
    # exercise the multi-rank plumbing on one GPU (NCCL ranks sharing a GPU
    # would wait on each other inside kernels)
    one_gpu = os.environ.get("FVR_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if one_gpu:
            torch.distributed.init_process_group("gloo")
        else:
            torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local))

    sc = make_scene()
    dev = torch.device("cuda", local)

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    stream = _lib.stream_ptr()

    def timed_loop(deterministic: bool, steps: int, warmup: int, sampler=None):
        """K timed iterations of one ChannelLoop, then K more with an event
        between every stage (the per-kernel breakdown the roofline uses).

        The timed pass is one event pair around the K steps: the loop's
        kernels chain through programmatic dependent launch, which an event
        between them would break.  No L2 flush: every step streams the two
        plans (0.75 GB at config 2) through a 126 MB L2."""
        cfg = ReconstructionConfig(alpha_l=ALPHA_L, alpha_d=1.0, tau=TAU, max_iters=2 * steps + warmup,
                                   converge_eps=1e-12, deterministic_mode=deterministic, g_sigma=0.1, rng_seed=0)
        grid0 = _init_grid(sc["geom"], sc["hull"], "green")
        src = [im.data[sc["bbox"].slices][:, :, 0] for im in sc["images"]]
        loop = ChannelLoop(sc["cams"], grid0, grid0.values, src, sc["masks"], sc["bbox"],
                           sc["hull"].inside_voxels(), sc["hull"].key_point_mask(), sc["rcfg"],
                           _loop_config(cfg, grid0), cfg.max_iters + 8, background=0.0, use_graph=False)
        stages = [(n, f) for n, f in loop.stages() if f is not None]
        names = [n for n, _ in stages]

        def one_step(evs=None):
            launches = 0
            if evs:
                evs[0].record()
            for i, (_, fn) in enumerate(stages):
                launches += fn(stream)
                if evs:
                    evs[i + 1].record()
            return launches

        def new_events():
            return [torch.cuda.Event(enable_timing=True) for _ in range(len(stages) + 1)]

        for _ in range(warmup):
            one_step()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        launches = 0
        # (NVTX range "timed": the launch list of exactly this region is
        # `ncu --nvtx --nvtx-include "timed/" ...`)
        torch.cuda.nvtx.range_push("timed")
        e0.record()
        for _ in range(steps):
            launches += one_step()
        e1.record()
        torch.cuda.nvtx.range_pop()
        barrier()
        timed_ms = e0.elapsed_time(e1)
        all_evs = []
        for _ in range(steps):  # the per-stage breakdown
            evs = new_events()
            one_step(evs)
            all_evs.append(evs)
        barrier()
        st = loop.read_state()
        assert st["it"] == warmup + 2 * steps and not st["done"], st
        return loop, names, all_evs, launches, grid0, src, timed_ms

    # clocks: sampled from before the first timed step to after the last
    # e2e call (the deterministic, stochastic and e2e regions)
    sampler = ClockSampler(local)
    sampler.start()
    sampler.wait_first()
    loop, names, all_evs, launches, grid0, src, total_ms = timed_loop(True, args.steps, args.warmup)
    part_ms = {n: float(np.mean([e[i].elapsed_time(e[i + 1]) for e in all_evs])) for i, n in enumerate(names)}
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())

    # the reference's default configuration draws a random G per sample
    # (deterministic_mode=False): same workload through the stochastic path
    stoch = None
    if args.stochastic_steps > 0:
        sl, snames, sevs, _, _, _, s_total = timed_loop(False, args.stochastic_steps, args.warmup)
        s_ms = s_total / args.stochastic_steps
        if world > 1:
            t = torch.tensor([s_ms], dtype=torch.float64, device=dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            s_ms = float(t.item())
        stoch = {"value": 1000.0 / s_ms, "unit": "iters/s", "ms_per_step": s_ms, "steps": args.stochastic_steps,
                 "stage_ms": {n: float(np.mean([e[i].elapsed_time(e[i + 1]) for e in sevs]))
                              for i, n in enumerate(snames)},
                 "adjust_path": ("sample-plan gather (nnz %d, %d sample slots, %s entries)"
                                 % (sl.plan_nnz, sl.n_samples, "6-byte" if sl.splan_e6 else "8-byte"))
                 if sl.plan else "ray-driven scatter",
                 "note": "deterministic_mode=False, g_sigma 0.1 (the reference default): per-sample Philox G"}
        del sl

    w = work_counts(sc)
    if loop.occ is not None:
        w["S_r_live"] = live_samples(sc, loop.occ)
    render_bytes, iter_bytes = algorithmic_bytes(w, scattering=True)
    ms = total_ms / args.steps
    its = 1000.0 / ms
    peak, peak_kind = peaks()
    render_ms = part_ms["render"]
    achieved = render_bytes / (render_ms * 1e-3) / 1e9
    live = w.get("S_r_live", w["S_r"])
    live_bytes = 108 * live + (w["S_r"] - live) + 8 * w["VP"]
    live_achieved = live_bytes / (render_ms * 1e-3) / 1e9
    if loop.rplan:
        kname = "rplan_render_kernel<1>"
        rows = loop.rp_len.numel() * 32
        # per row: base (8 B) unless the loop started from its own lattice, t_fin (8 B) for a nonzero background
        row_b = (0 if loop._static_zero else 8) + (8 if any(b != 0.0 for b in loop.background) else 0)
        kbytes = 6 * loop.rplan_nnz + row_b * rows + 8 * w["VP"]
        rule = (f"render plan: 6 B per stored SELL entry (24-bit key-point index + 24-bit weight) + {row_b} B per "
                "row (base f64 unless the loop starts from its own lattice, t_fin f64 for a nonzero background) + "
                "8 B per bbox pixel (src in, residual out); the key-point operand (1.2 MB) hits L1/L2")
    else:
        kname = "loop_render_scat_kernel"
        kbytes = live_bytes
        rule = "108 B per live sample + 1 B per skipped sample + 8 B per bbox pixel (marching kernel)"
    kach = kbytes / (render_ms * 1e-3) / 1e9
    roof = {"bound": "hbm", "kernel": kname, "achieved": kach, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
            "frac": kach / peak, "traffic": TRAFFIC_BYTES_PER_LAUNCH[kname], "traffic_source": TRAFFIC_SOURCE[kname],
            "bytes_per_launch": kbytes, "bytes_rule": rule,
            # the render only reads (516 MB in, ~1 MB out): the read-only stream ceiling next to the copy peak
            "read_stream_peak": {"gbs": READ_STREAM_GBS, "frac": kach / READ_STREAM_GBS, "source": READ_STREAM_SOURCE}}

    # What one step streams from HBM (the plans are re-read every iteration;
    # the operands they index are cache-resident): render plan (6 B per stored
    # entry + base/t_fin per row as streamed + 8 B per pixel) and adjust plan (6 B per stored
    # entry + 20 B per hull key point: row order, key-point index, value
    # read/write, operand write)
    adj_bytes = 6 * loop.plan_slots + 20 * loop.n_kp if loop.plan else 0
    step_bytes = kbytes + adj_bytes
    step_streamed = {"bytes": step_bytes, "render_bytes": kbytes, "adjust_bytes": adj_bytes,
                     "achieved_gbs": step_bytes / (ms * 1e-3) / 1e9, "frac": step_bytes / (ms * 1e-3) / 1e9 / peak,
                     "rule": "render plan 6 B/stored entry + base/t_fin as streamed + 8 B/pixel; adjust plan 6 B/stored entry + "
                             "20 B/hull key point; over the whole step time (both launches + gaps)"}
    # Per-call model of the public API: the plans are built once per
    # reconstruct_channel call (count + fill passes over every ray), then
    # streamed every iteration
    plan_bytes = 6 * loop.rplan_nnz + 16 * (loop.rp_len.numel() * 32 if loop.rplan else 0) + \
        (6 * loop.plan_slots if loop.plan else 0)
    per_call = {"plan_bytes_written": plan_bytes, "step_ms": ms}

    # e2e: the public API with host buffers (H2D of inputs, D2H of the grid)
    e2e = None
    if args.e2e_iters > 0:
        cfg_e = ReconstructionConfig(alpha_l=ALPHA_L, alpha_d=1.0, tau=TAU, max_iters=args.e2e_iters,
                                     converge_eps=1e-12, deterministic_mode=True)
        reconstruct_channel(sc["images"], sc["cams"], sc["geom"], sc["hull"], cfg_e, render_cfg=sc["rcfg"],
                            masks=sc["masks"], bbox=sc["bbox"])  # warm (graph capture path, allocator)
        walls = []
        prof = None
        if os.environ.get("FVR_E2E_PROFILE"):
            import cProfile

            prof = cProfile.Profile()
        for _ in range(9):  # median of nine calls (~11 ms each; the clock sampler's 100 ms nvidia-smi query stalls one or two)
            barrier()
            if prof:
                prof.enable()
            t0 = time.perf_counter()
            grid, trace = reconstruct_channel(sc["images"], sc["cams"], sc["geom"], sc["hull"], cfg_e,
                                              render_cfg=sc["rcfg"], masks=sc["masks"], bbox=sc["bbox"])
            barrier()
            walls.append(time.perf_counter() - t0)
            if prof:
                prof.disable()
        if prof:
            import pstats

            pstats.Stats(prof, stream=sys.stderr).sort_stats("tottime").print_stats(15)
        wall = float(np.median(walls))
        if world > 1:
            t = torch.tensor([wall], dtype=torch.float64, device=dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            wall = float(t.item())
        # what reconstruct_channel copies: the bbox crops of the frames (f32)
        # and of the masks (u8), the inside-voxel bytes and the camera
        # structs in; the lattice and the trace out (hull key points, the
        # initial lattice and the flame-ray list are derived on the device)
        bb = sc["bbox"]
        h2d = (sum(s.nbytes for s in src) + N_VIEWS * bb.area + sc["hull"].inside_voxels().size
               + ctypes.sizeof(_lib.FvrCamera) * N_VIEWS)
        d2h = grid.values.nbytes + 8 * trace.iterations
        # the call = setup (host staging, uploads, hull key points, both plans'
        # count + fill passes) + the iterations + the result copy
        per_call.update(call_ms=wall * 1e3, iterations_ms=trace.iterations * ms,
                        setup_and_io_ms=wall * 1e3 - trace.iterations * ms,
                        plan_write_gbs=plan_bytes / max(wall - trace.iterations * ms * 1e-3, 1e-9) / 1e9,
                        note="setup_and_io = call - iterations x the timed step (cold-L2 step time, so an "
                             "upper bound on the iterations' share); the plans are written once per call")
        e2e = {"value": trace.iterations / wall, "unit": "iters/s", "iterations": trace.iterations,
               "h2d_bytes_per_step": int(h2d / trace.iterations), "d2h_bytes_per_step": int(d2h / trace.iterations),
               "calls_ms": [1e3 * x for x in walls],
               "note": "reconstruct_channel() on host numpy inputs; H2D of frames/lattice/hull and D2H of the "
                       "grid + trace inside the timed call, amortised over its iterations; median of 9 calls"}
        if stoch is not None:
            # the same public call in the reference's default mode (per-sample random G)
            cfg_s = ReconstructionConfig(alpha_l=ALPHA_L, alpha_d=1.0, tau=TAU, max_iters=args.e2e_iters,
                                         converge_eps=1e-12, deterministic_mode=False, g_sigma=0.1, rng_seed=0)
            s_walls = []
            for i in range(6):
                barrier()
                t0 = time.perf_counter()
                _, s_trace = reconstruct_channel(sc["images"], sc["cams"], sc["geom"], sc["hull"], cfg_s,
                                                 render_cfg=sc["rcfg"], masks=sc["masks"], bbox=sc["bbox"])
                barrier()
                if i:  # the first call warms the sample-plan path
                    s_walls.append(time.perf_counter() - t0)
            s_wall = float(np.median(s_walls))
            stoch["e2e"] = {"value": s_trace.iterations / s_wall, "unit": "iters/s", "iterations": s_trace.iterations,
                            "calls_ms": [1e3 * x for x in s_walls],
                            "note": "reconstruct_channel(deterministic_mode=False) from host arrays, median of 5 "
                                    "calls; rank-local wall time"}

    time.sleep(0.15)  # one more nvidia-smi row after the last timed region
    clocks = sampler.stop()
    out = {
        "metric": METRIC,
        "value": its,
        "unit": "iters/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": DTYPE,
        "data": "synthetic (synth_volume seed 0, synth_cameras seed 0, inputs rendered on device)",
        "config": workloads.bench_config(N_VOX, N_VIEWS, RES, (sc["bbox"].u0, sc["bbox"].v0, sc["bbox"].u1,
                                                               sc["bbox"].v1), world),
        "gsamples_per_s": (w["S_r"] + w["S_a"]) * its / 1e9,
        "render_gsamples_per_s": w["S_r"] / (render_ms * 1e-3) / 1e9,
        "work": w,
        "stage_ms": part_ms,
        # the SURVEY 8(d) per-iteration bytes of the reference's work (what a
        # marching implementation would move); the plans make the step move
        # far less, so this is a work rate, not an HBM fraction
        "iter_survey_bytes": iter_bytes,
        "step_streamed": step_streamed,
        "per_call": per_call,
        # Dominant kernel = K-render.  Through the render plan it streams B
        # (6 B per stored SELL entry, padding included) plus per-row base and
        # t_fin (16 B) and src/residual (8 B per pixel); the key-point operand
        # it multiplies is cache-resident.
        "roofline": roof,
        "roofline_survey_rule": {"bytes_per_launch": live_bytes, "achieved": live_achieved,
                                 "frac": live_achieved / peak,
                                 "rule": "SURVEY 8(d) per-sample figure: 108 B per live sample + 1 B per skipped "
                                         "sample + 8 B per bbox pixel, over the same K-render time"},
        "roofline_dense_equiv": {"bytes_per_launch": render_bytes, "achieved": achieved, "frac": achieved / peak,
                                 "rule": "108 B for every render sample S_r as if none were skipped (the "
                                         "reference's work), over the same K-render time"},
        "gpu_launches": int(launches),
        "render_path": ("render plan (SELL-32, %d stored entries)" % loop.rplan_nnz) if loop.rplan
        else "marching kernel",
        "adjust_path": ("voxel-driven gather (SELL-32 plan, nnz %d, %d stored)" % (loop.plan_nnz, loop.plan_slots))
        if loop.plan else "ray-driven scatter",
        "clocks": clocks,
        "stochastic": stoch,
        "e2e": e2e,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(sc, args.cpu_seconds)
    if rank == 0:
        print(json.dumps(out))
    if world > 1:
        torch.distributed.destroy_process_group()


# ---------------------------------------------------------------------------
# CPU oracle (reference arm and cpu_baseline)
# ---------------------------------------------------------------------------


def _oracle_iteration_sample(sc, values, views, cpu):
    """Render + adjust of the given views of one iteration on the CPU oracle."""
    geom, bbox = sc["geom"], sc["bbox"]
    u0, v0, u1, v1 = bbox.u0, bbox.v0, bbox.u1, bbox.v1
    uu, vv = np.meshgrid(np.arange(u0, u1 + 1) + 0.5, np.arange(v0, v1 + 1) + 0.5, indexing="xy")
    inside = sc["hull"].inside_voxels()
    residuals = []
    for v in views:
        cam = sc["cams"][v]
        rec = cpu.render_pixels(cam, values[None], geom.origin, geom.edge, TAU, 1.0, np.zeros(1), uu.ravel(),
                                vv.ravel(), scattering=True, sigma_s=SIGMA_S, scatter_dirs=SCAT_DIRS)
        src = sc["images"][v].data[bbox.slices][:, :, 0].astype(np.float64)
        f = np.zeros((cam.height, cam.width))
        f[v0:v1 + 1, u0:u1 + 1] = src - rec.reshape(src.shape)
        residuals.append(f)
    alpha_d_eff = 1.0 * (0.2 / float(np.max(geom.box.size)))
    return cpu.adjust_pass(values, inside, [sc["cams"][v] for v in views], residuals,
                           [sc["masks"][v].bits for v in views], (u0, v0, u1, v1), geom.origin, geom.edge, TAU,
                           ALPHA_L, alpha_d_eff)


def cpu_baseline(sc, budget_s):
    from oracle import cpu

    cores = os.cpu_count() or 1
    cpu.set_threads(cores)
    values = sc["geom"].copy().values
    from paper_1809_06417_b200.reconstruct import _init_grid

    values = _init_grid(sc["geom"], sc["hull"], "green").values
    n_done, t_total = 0, 0.0
    views = list(range(N_VIEWS))
    while t_total < budget_s and n_done < 3:
        t0 = time.perf_counter()
        values = _oracle_iteration_sample(sc, values, views, cpu)
        t_total += time.perf_counter() - t0
        n_done += 1
    return {"value": n_done / t_total, "unit": "iters/s", "cores": cores, "kind": "port",
            "sample": f"{n_done} full iteration(s) of the workload (8 views render w/ scattering + adjust) "
                      f"on the C/OpenMP oracle, {t_total:.1f} s",
            "cpu": _cpu_model()}


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def run_reference(args):
    """The reference arm: the unmodified reference package (baseline/_ref,
    numba kernels on the host cores) through its own public API, on the same
    workload and config as the GPU arm.  The scene is built by the reference
    itself (workloads.reference_scene); this package and its library are never
    imported.  A step is ``views_per_step`` views of one loop iteration
    (reconstruct.py:304-331): render_pixels of each view's bbox pixels, the
    per-view RMSE and residual field, then one adjust_pass over those views;
    views_per_step is sized from a timed warm-up so that the whole --steps K
    --warmup W run stays within a few minutes.  iters/s = views_per_step /
    (V * mean step time)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    if rank != 0:
        return
    import workloads

    if not workloads.reference_available():
        print(json.dumps({"impl": "reference", "unavailable": "baseline/_ref is not installed (see DESIGN.md §6 for "
                                                              "the pip --target install of /root/reference/pkg)"}))
        return
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    sc = workloads.reference_scene(N_VOX, N_VIEWS, RES)
    scene_s = time.perf_counter() - t0
    ref = sc["ref"]
    R = ref["reconstruct"]
    cfg = R.ReconstructionConfig(alpha_l=ALPHA_L, alpha_d=1.0, tau=TAU, max_iters=args.steps + args.warmup,
                                 converge_eps=1e-12, deterministic_mode=True)
    grid = R._init_grid(sc["geom"], sc["hull"], "green")
    rng = np.random.default_rng(cfg.rng_seed)
    b = sc["bbox"]
    h_bb, w_bb = b.v1 - b.v0 + 1, b.u1 - b.u0 + 1
    uu, vv = np.meshgrid(np.arange(b.u0, b.u1 + 1, dtype=np.float64) + 0.5,
                         np.arange(b.v0, b.v1 + 1, dtype=np.float64) + 0.5, indexing="xy")
    us, vs = uu.ravel(), vv.ravel()
    src = [im.data[b.slices][:, :, 0].astype(np.float64) for im in sc["images"]]

    def step(views):
        residuals = []
        for v in views:
            cam = sc["cams"][v]
            rec = ref["render"].render_pixels(cam, [grid], sc["rcfg"], us, vs).reshape(h_bb, w_bb)
            float(np.sqrt(np.mean((src[v] - rec) ** 2)))
            field = np.zeros((cam.height, cam.width))
            field[b.slices] = src[v] - rec
            residuals.append(field)
        R.adjust_pass(grid, sc["hull"], [sc["cams"][v] for v in views], residuals, [sc["masks"][v] for v in views],
                      cfg, rng, b)

    t0 = time.perf_counter()
    step([0])  # numba JIT of render_rays / adjust_rays_chunked, then one timed view
    jit_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    step([1 % N_VIEWS])
    per_view = time.perf_counter() - t0
    n_steps = args.steps + args.warmup
    views_per_step = int(max(1, min(N_VIEWS, args.reference_seconds / max(per_view * n_steps, 1e-9))))
    times = []
    for s in range(n_steps):
        views = [(s * views_per_step + i) % N_VIEWS for i in range(views_per_step)]
        t0 = time.perf_counter()
        step(views)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            times.append(dt)
    per_step = float(np.mean(times))
    its = views_per_step / (N_VIEWS * per_step)
    sample = (f"each step = {views_per_step} of {N_VIEWS} views of one iteration through the reference's public API "
              f"(fvr.render.render_pixels of the view's bbox pixels with scattering + fvr.reconstruct.adjust_pass), "
              f"numba on {cores} host threads; iters/s = views_per_step / ({N_VIEWS} * step time); scene built by "
              f"the reference in {scene_s:.0f} s, JIT warm-up {jit_s:.0f} s")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": its, "unit": "iters/s", "n_gpus": world,
        "device": "host cores only (the reference path is CPU code)",
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_step * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64 geometry and accumulation, f32 lattice",
        "data": "synthetic (synth_volume seed 0, synth_cameras seed 0, inputs rendered by the reference)",
        "config": workloads.bench_config(N_VOX, N_VIEWS, RES, (b.u0, b.v0, b.u1, b.v1), world),
        "cpu_baseline": {"value": its, "unit": "iters/s", "cores": cores, "kind": "reference", "sample": sample,
                         "cpu": _cpu_model()},
        "e2e": {"value": its, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--e2e-iters", type=int, default=50)
    ap.add_argument("--stochastic-steps", type=int, default=20)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--reference-seconds", type=float, default=120.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: relaunch under torchrun (rank 0 prints the line)
        import socket

        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
