"""Device-resident reconstruction loop (one scalar channel, or three).

One iteration of reconstruct_channel (reconstruct.py:304-334) is two
launches on one stream (deterministic mode; the stochastic mode adds a
weigh launch between them):

  K-render   the render plan B (SELL-32, csrc/fvr_rplan.cuh): every bbox
             pixel's row of B times the hull key-point values, plus its
             static base and t_fin * background; residual and squared-
             residual partials; the last CTA finalizes the iteration (per-
             view RMSE, mean, trace append, convergence rule, done flag)
  K-adjust   the adjust plan A (SELL-32 gather by hull key point,
             csrc/fvr_plan.cu): every hull key point sums its weighted
             residuals in 32.32 fixed point and updates its value,
             v = f32(max(v + delta, -1)), skipped when the rule fired

Both plans are built once per call on the device from the geometry (count
pass, scan, fill).  Hull key points are renumbered in Morton order so both
operands stay L2-local.  The reference's break-before-adjust holds because
the adjust reads the done flag the render's finalize wrote; once ``done`` is
set every later launch is a no-op, so the host enqueues iterations (or
replays a captured CUDA graph) without a per-iteration round trip and reads
the trace back at the end.  Where a plan cannot be built (device memory) the
loop uses the marching kernels (csrc/fvr_render.cu, csrc/fvr_adjust.cu) on
the same contract.

With a process group (world_size > 1) the views are sharded in contiguous
ranges across ranks; each rank renders and back-projects its own views and
one all-reduce per iteration of an int64 buffer [packed correction at hull
key points | squared-residual partials of every view] -- NCCL behind the
C ABI (fvr_comm_init / fvr_allreduce_sum, csrc/fvr_comm.cu) on CUDA, gloo in
the CPU tests -- makes every rank's lattice identical.  Integer sums are
exact, so 1, 2, 4 or 8 GPUs give bit-identical grids.
"""

from __future__ import annotations

import ctypes
import os
import time
from dataclasses import dataclass

import numpy as np

from . import _lib


@dataclass
class LoopConfig:
    tau: float
    alpha_l: float
    alpha_d_eff: float
    converge_eps: float
    stochastic: bool
    g_sigma: float
    seed: int


def _world():
    """(rank, world_size, sharded): sharded when torch.distributed is
    initialised with more than one rank (or FVR_FORCE_SHARDED=1, which runs the
    exchange path on a 1-rank group -- used to test it on one GPU)."""
    if os.environ.get("FVR_NO_SHARDING") == "1":
        return 0, 1, False
    t = _lib.torch()
    if t.distributed.is_available() and t.distributed.is_initialized():
        rank, world = t.distributed.get_rank(), t.distributed.get_world_size()
        return rank, world, world > 1 or os.environ.get("FVR_FORCE_SHARDED") == "1"
    return 0, 1, False


def shard_views(n_views: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced view range [begin, end) of one rank."""
    base, extra = divmod(n_views, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


class DeviceComm:
    """The data-path collective behind the C ABI: an ncclComm_t owned by
    libfvr_b200 (fvr_comm_init / fvr_allreduce_sum / fvr_comm_destroy), one per
    process group.  torch.distributed only carries the 128-byte unique id
    (a broadcast over the group's store-backed rendezvous)."""

    _cache: dict = {}

    def __init__(self, group=None):
        import torch.distributed as dist

        t = _lib.torch()
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        uid = (ctypes.c_uint8 * _lib.FVR_COMM_ID_BYTES)()
        if self.rank == 0:
            _lib.call("fvr_comm_unique_id", ctypes.addressof(uid))
        box = [bytes(uid)]
        dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group is not None else 0,
                                   group=group)
        uid = (ctypes.c_uint8 * _lib.FVR_COMM_ID_BYTES).from_buffer_copy(box[0])
        self.handle = ctypes.c_void_p()
        _lib.call("fvr_comm_init", self.rank, self.world, ctypes.addressof(uid), t.cuda.current_device(),
                  ctypes.byref(self.handle))

    @classmethod
    def for_group(cls, group=None) -> "DeviceComm":
        import torch.distributed as dist

        key = (id(group), dist.get_rank(group), dist.get_world_size(group))
        if key not in cls._cache:
            cls._cache[key] = cls(group)
        return cls._cache[key]

    def allreduce_sum_(self, buf, stream) -> None:
        dt = {"torch.int64": _lib.FVR_DT_INT64, "torch.float32": _lib.FVR_DT_FLOAT32,
              "torch.float64": _lib.FVR_DT_FLOAT64}[str(buf.dtype)]
        _lib.call("fvr_allreduce_sum", self.handle, buf.data_ptr(), buf.numel(), dt, stream)


def _collective(group=None):
    """The exchange's transport: the library's own NCCL communicator when the
    process group runs NCCL (the production path), torch.distributed
    otherwise (gloo: the CPU tests and the one-GPU multi-process test, whose
    ranks must not run kernels that wait on each other)."""
    import torch.distributed as dist

    if dist.get_backend(group) == "nccl" and os.environ.get("FVR_TORCH_COLLECTIVE") != "1":
        return DeviceComm.for_group(group)
    return None


def exchange(comm, sq, vol, v_begin: int, v_end: int, rows_per_view: int, rank: int, group=None,
             stream=None) -> None:
    """The one collective of an iteration (§8e): all-reduce(sum) of the i64
    buffer ``comm`` = [packed correction | squared-residual partials (f64 bits)
    | volume partials (f64 bits)] across the ranks of ``group``.

    Corrections are 32.32 fixed-point integers, so their sum is exact and
    independent of the partition.  Each f64 partial has exactly one owner
    (the rank of its view; rank 0 for the replicated volume term): all other
    ranks contribute the bit pattern of +0.0, i.e. integer 0, so the integer
    sum reproduces the owner's bits exactly.  ``sq``/``vol`` are f64 views into
    ``comm`` (``sq`` may carry a leading channel axis).  CUDA tensors under an
    NCCL group go through fvr_allreduce_sum on ``stream``; CPU tensors (gloo)
    through torch.distributed.
    """
    import torch.distributed as dist

    sq[..., : v_begin * rows_per_view].zero_()
    sq[..., v_end * rows_per_view:].zero_()
    if vol is not None and rank != 0:
        vol.zero_()
    dc = _collective(group) if comm.is_cuda else None
    if dc is not None:
        dc.allreduce_sum_(comm, _lib.stream_ptr() if stream is None else stream)
    else:
        dist.all_reduce(comm, op=dist.ReduceOp.SUM, group=group)


_SIDE: dict = {}
_SCAT: dict = {}


def _scatter_dirs(n: int, dev):
    """fibonacci_sphere(n) on the device, built once per (n, device)."""
    key = (n, str(dev))
    if key not in _SCAT:
        from .radiometry import fibonacci_sphere

        _SCAT[key] = _lib.torch().from_numpy(np.ascontiguousarray(fibonacci_sphere(n))).to(dev)
    return _SCAT[key]


def _side_stream(dev):
    """One persistent side stream per device: buffers allocated on it come
    from its own caching-allocator pool, which a per-call stream would never
    reuse (a fresh cudaMalloc every call)."""
    t = _lib.torch()
    # higher priority than the loop's stream (FVR_SIDE_PRIORITY, default -1):
    # the side stream's short layout kernels are scheduled ahead of a running
    # fill's remaining CTAs instead of after them
    prio = int(os.environ.get("FVR_SIDE_PRIORITY", "-1"))
    key = (str(dev), prio)
    if key not in _SIDE:
        _SIDE[key] = t.cuda.Stream(device=dev, priority=prio)
    return _SIDE[key]


_PINNED: dict = {}


def _pinned_ring(shape, dtype, depth):
    """Page-locked host buffers for the snapshot ring, kept for the process
    (cudaHostAlloc costs milliseconds; snapshots of one shape reuse them)."""
    key = (shape, dtype, depth)
    if key not in _PINNED:
        t = _lib.torch()
        _PINNED[key] = [t.empty(shape, dtype=dtype, pin_memory=True) for _ in range(depth)]
    return _PINNED[key]


# Hull key points are numbered in Morton (x, y, z) order: the render plan's
# operand and the adjust plans' rows follow that numbering, so the key points
# of a 2x2x2 block are neighbours in memory (config 2: K-render 0.1015 ->
# 0.0995 ms, K-adjust 0.0636 -> 0.0607, stochastic sample-plan gather 0.153 ->
# 0.114).  FVR_KP_ORDER=lattice keeps the lattice order.
def _morton_enabled() -> bool:
    return os.environ.get("FVR_KP_ORDER", "morton") != "lattice"


def _nonzero_u8(mask):
    """Indices (int32, device) of the nonzero bytes of ``mask``: a native
    count, one synchronisation for the size, a native select."""
    t = _lib.torch()
    flat = mask.reshape(-1)
    n = int(flat.numel())
    cnt = t.empty(1, dtype=t.int64, device=flat.device)
    _lib.call("fvr_count_nonzero_u8", flat.data_ptr(), n, cnt.data_ptr(), _lib.stream_ptr())
    m = int(cnt.item())
    out = t.empty(m, dtype=t.int32, device=flat.device)
    if m:
        _lib.call("fvr_select_nonzero_u8", flat.data_ptr(), n, m, out.data_ptr(), cnt.data_ptr(), _lib.stream_ptr())
    return out


def _morton_order(kp, shape):
    """The list of lattice indices ``kp`` (int32, device) sorted by Morton
    (x, y, z) code: one key kernel and one radix sort over the code's bits
    (fvr_morton_order)."""
    t = _lib.torch()
    n = int(kp.numel())
    if n == 0:
        return kp
    out = t.empty_like(kp)
    g = _lib.FvrGrid()
    g.nx, g.ny, g.nz = shape[0] - 1, shape[1] - 1, shape[2] - 1
    g.edge = 1.0
    _lib.call("fvr_morton_order", kp.contiguous().data_ptr(), n, g, out.data_ptr(), _lib.stream_ptr())
    return out


class ChannelLoop:
    """Owns the device buffers of one reconstruct_channel call -- or of the
    three channels of reconstruct_color batched into one loop (values of
    shape (3, *lattice), src (3, V, h, w), backgrounds per channel): the
    channels share rays, hull, plan and launches, and each keeps its own
    convergence state (a converged channel is frozen while the others go on).
    """

    def __init__(self, cameras, grid_geom, values, src_blocks, masks, bbox, inside, kp_mask,
                 render_cfg, loop_cfg: LoopConfig, max_iters: int, ground_truth=None,
                 background=0.0, use_graph: bool = True, n_channels: int = 1, mask_crops=None):
        t = _lib.torch()
        self.t = t
        self.dev = _lib.device()
        self.rank, self.world, self.sharded = _world()
        if n_channels not in (1, 3):
            raise ValueError("the loop runs 1 or 3 channels")
        C = self.nch = int(n_channels)
        V = len(cameras)
        self.n_views = V
        self.v_begin, self.v_end = shard_views(V, self.rank, self.world)
        local = list(range(self.v_begin, self.v_end))
        self.bbox = bbox
        self.w_bb, self.h_bb = bbox.u1 - bbox.u0 + 1, bbox.v1 - bbox.v0 + 1
        self.grid = _lib.grid_struct(grid_geom)
        self.cfg = loop_cfg
        self.max_iters = int(max_iters)
        dev = self.dev

        # FVR_INIT_PROFILE=1: host time and device events at section marks
        self._marks = [] if os.environ.get("FVR_INIT_PROFILE") == "1" else None
        self._mark("start")
        # geometry and inputs
        self.cams = _lib.cameras_tensor([cameras[v] for v in local], dev) if local else None
        if t.is_tensor(src_blocks):  # ([C,] V, h, w) f32 device crops (DeviceFrames)
            blk = src_blocks if src_blocks.dim() == 4 else src_blocks.unsqueeze(0)
            self.src = blk[:, self.v_begin:self.v_end].contiguous() if local else \
                t.zeros((C, 1, 1, 1), dtype=t.float32, device=dev)
        else:
            arr = np.stack([src_blocks[v] for v in local]) if local else np.zeros((1, 1, 1), np.float32)
            arr = arr[None] if C == 1 else np.moveaxis(arr, -1, 0)
            self.src = t.from_numpy(np.ascontiguousarray(arr, dtype=np.float32)).to(dev)
        if self.src.shape[0] != C:
            raise ValueError("src channels do not match n_channels")
        shape = (grid_geom.nx + 1, grid_geom.ny + 1, grid_geom.nz + 1)
        self.shape = shape
        if t.is_tensor(inside):  # u8 (nx, ny, nz), staged on the device already
            self.inside = inside
        else:
            inside = np.ascontiguousarray(inside)
            if inside.dtype == np.bool_:  # upload the bytes as they are (no host-side u8 copy)
                self.inside = t.from_numpy(inside).to(dev).view(t.uint8)
            else:
                self.inside = t.from_numpy(inside.astype(np.uint8)).to(dev)
        self._mark("cams+src+inside")
        self.values = t.empty((C,) + shape, dtype=t.float32, device=dev)
        if values is not None:
            self.values.copy_(t.from_numpy(np.ascontiguousarray(values, dtype=np.float32)).reshape((C,) + shape))
        # the loop's own initial lattice (0 on hull key points, -1 elsewhere)
        # has no positive key point outside the hull: the render plan's base
        # then needs no static term (no pos27 pass)
        self._static_zero = values is None
        if kp_mask is None or values is None:
            # hull key points (and the initial lattice when values is None)
            # derived on the device from the inside voxels
            kp_dev = t.empty(shape, dtype=t.uint8, device=dev)
            _lib.call("fvr_hull_keypoints", self.inside.data_ptr(), self.grid, kp_dev.data_ptr(),
                      self.values.data_ptr() if values is None else None, _lib.stream_ptr())
            if values is None and C > 1:
                self.values[1:].copy_(self.values[0:1].expand((C - 1,) + shape))
            if kp_mask is not None:
                kp_dev = t.from_numpy(np.ascontiguousarray(kp_mask, dtype=np.uint8)).to(dev)
            self.kp = None  # listed below, after the work that needs only kp_dev is enqueued
        else:
            kp_dev = t.from_numpy(np.ascontiguousarray(kp_mask, dtype=np.uint8)).to(dev)
            kp_idx = np.flatnonzero(kp_mask.ravel()).astype(np.int32)
            self.n_kp = int(kp_idx.size)
            self.kp = t.from_numpy(kp_idx if kp_idx.size else np.zeros(1, np.int32)).to(dev)
            if _morton_enabled() and self.n_kp:
                self.kp = _morton_order(self.kp, shape)
        self.accum = None  # scatter path only
        kp_ready = t.cuda.Event()  # kp_dev (and the initial lattice) on the loop's stream
        kp_ready.record()

        self._mark("inputs+hull kp")
        # render configuration of the loop (render_pixels without a phase: g = 0)
        self.scattering = bool(render_cfg.scattering_enabled and render_cfg.sigma_s > 0.0)
        if self.scattering:
            self.scat = _scatter_dirs(int(render_cfg.scatter_dirs), dev)
            n_scat = int(self.scat.shape[0])
        else:
            self.scat = None
            n_scat = 1
        self.params = _lib.render_params(render_cfg, self.scattering, n_scat, 0.0, grid_geom.edge)
        bg = np.broadcast_to(np.asarray(background, dtype=np.float64).reshape(-1), (C,))
        self.background = (ctypes.c_double * C)(*[float(x) for x in bg])
        # packed copy of max(v, 0) read by the marching render, kept in sync by
        # K-update; packed once the plans are decided (the render plan reads
        # its own operand, so with it the layout is neither built nor updated)
        self.layout_kind = _lib.layout_kind(self.params, self.grid)
        self.layout = None
        # empty-space occupancy: hull key points (their values change) plus any
        # positive initial value of any channel; key points outside the hull are
        # never written, so the map stays valid for the whole loop
        self.occ = None
        if self.layout_kind and os.environ.get("FVR_NO_SKIP") != "1":
            self.occ = t.empty(shape, dtype=t.uint8, device=dev)
            _lib.call("fvr_occupancy", self.values.data_ptr(), C, kp_dev.data_ptr(), self.grid,
                      self.occ.data_ptr(), _lib.stream_ptr())
        self.kp_dev = kp_dev

        self.bpv = int(_lib.load().fvr_loop_blocks_per_view(self.w_bb, self.h_bb))
        self.rplan = False
        self.rplan_nnz = 0
        self._rp_counted = None
        self._mark("layout+occupancy")
        # flame rays of the local views, row-major per view (reconstruct.py:144-149)
        # compacted on the device (host masks: the bbox crops are uploaded)
        n_host = None
        if mask_crops is not None:  # (V, h, w) u8 device crops + host flame counts per view
            sub, per_view = mask_crops
            n_host = int(per_view[self.v_begin:self.v_end].sum())
        elif t.is_tensor(masks):  # (V, H, W) u8 device masks
            sub = masks[:, bbox.v0:bbox.v1 + 1, bbox.u0:bbox.u1 + 1]
        else:
            crops = np.stack([np.asarray(masks[v].bits[bbox.slices], dtype=np.uint8) for v in range(V)])
            per_view = np.count_nonzero(crops.reshape(V, -1), axis=1)
            n_host = int(per_view[self.v_begin:self.v_end].sum())
            sub = t.from_numpy(crops).to(dev)
        ray_base = 0
        if self.v_begin > 0:
            ray_base = int(per_view[: self.v_begin].sum()) if n_host is not None else \
                int(sub[: self.v_begin].reshape(-1).count_nonzero().item())
        local_sub = sub[self.v_begin:self.v_end]
        if local_sub.dtype != t.uint8:
            local_sub = local_sub.to(t.uint8)
        local_sub = local_sub.contiguous()
        if n_host is None:  # device masks: count them (one synchronisation)
            cnt = t.empty(1, dtype=t.int64, device=dev)
            _lib.call("fvr_count_nonzero_u8", local_sub.data_ptr(), local_sub.numel(), cnt.data_ptr(),
                      _lib.stream_ptr())
            n_host = int(cnt.item())
        # one native compaction (rows in view, row, col order)
        ray_list_t = t.empty(n_host, dtype=t.int32, device=dev)
        n_found = t.empty(1, dtype=t.int64, device=dev)
        if n_host:
            _lib.call("fvr_flame_rays", local_sub.data_ptr(), self.v_end - self.v_begin, self.w_bb, self.h_bb,
                      n_host, ray_list_t.data_ptr(), n_found.data_ptr(), _lib.stream_ptr())
        self.n_rays = int(ray_list_t.numel())
        self.rays = ray_list_t if self.n_rays else t.zeros(1, dtype=t.int32, device=dev)
        self.ray_base = ray_base
        # the render plan's count pass needs only the geometry, the occupancy
        # and kp_dev: it is queued on the loop's stream before anything waits
        # on the host; the hull key-point list (whose count the host must
        # read) and later the adjust plan's count are built on a persistent
        # side stream meanwhile
        main = t.cuda.current_stream()
        side = _side_stream(dev)
        pre = t.cuda.Event()
        pre.record(main)
        if self.layout_kind and os.environ.get("FVR_RENDER", "plan") != "march":
            self._rp_counted = self._rplan_count()
        self._mark("render count queued")
        side.wait_event(kp_ready)  # (the key-point list does not wait for the occupancy)
        if self.kp is None:
            with t.cuda.stream(side):
                kp_t = _nonzero_u8(kp_dev)  # synchronises the side stream
                if _morton_enabled():  # only the key-point list is ordered (no lattice-sized permutation)
                    kp_t = _morton_order(kp_t, shape)
            self.n_kp = int(kp_t.numel())
            self.kp = kp_t if self.n_kp else t.zeros(1, dtype=t.int32, device=dev)
            self.kp.record_stream(main)
            main.wait_stream(side)  # (later work on the loop's stream reads the list)
        self._mark("kp list")
        side.wait_event(pre)  # the flame rays, for the adjust plan's count
        if self.n_rays > 0 and self.n_kp > 0 and os.environ.get("FVR_ADJUST") != "scatter":
            with t.cuda.stream(side):  # the key-point map both plan fills read
                self._kp_map()
                self._kpmap.record_stream(main)
        self._mark("kp map")
        # channels interleaved per pixel (pitch 1, or 4 for three channels)
        self.pitch = 1 if C == 1 else 4
        # K-adjust as a voxel-driven gather over a precomputed plan: the merged
        # operator A in deterministic mode, the per-sample plan (weights G
        # applied through rho each iteration) in stochastic mode; the
        # ray-driven scatter remains for plans that would not fit
        self.plan = (self.n_rays > 0 and self.n_kp > 0 and os.environ.get("FVR_ADJUST") != "scatter")
        self.sample_plan = self.plan and loop_cfg.stochastic
        self.plan_nnz = 0
        self.n_samples = 0
        self.splan_e6 = False
        self.rho = None
        self._mark("plan flags")
        # The plan builds on two streams.  The render plan's count pass was
        # queued on the loop's stream above, so its layout and fill go first
        # there (the fill waits only for the key-point map); the adjust plan's
        # map, count pass and layout run on the side stream meanwhile, and its
        # fill runs beside the render plan's (the side stream has the higher
        # priority).  Once both fills were trimmed (register-staged chunk
        # stores, 4-5 CTAs per SM) the overlap pays: config 2 call 10.23 ->
        # 10.11 ms, stochastic 14.47 -> 14.26 ms (tools/e2e_ab.py); earlier
        # fills slowed each other.  FVR_FILL_SERIAL=1 runs them in sequence.
        keep = []
        adjust_done = kpmap_ready = pc = None
        rs = self._rplan_scan(*self._rp_counted) if self._rp_counted is not None else None
        self._rp_counted = None
        if rs is not None:  # the sizes leave as soon as the layout is done
            rs["sizes"] = _lib.HostRead(rs["sizes"])
        self._mark("render layout queued")
        if self.plan:
            kpmap_ready = t.cuda.Event()
            kpmap_ready.record(side)
            with t.cuda.stream(side):  # queued ahead of the render fill, which would hold every SM
                pc = self._plan_count()
                pc["sizes"] = _lib.HostRead(pc["sizes"])
        self._mark("adjust count queued")
        rfill_done = None
        if rs is not None:
            sizes = rs["sizes"].get()
            self._mark("render sizes read")
            if kpmap_ready is not None:
                main.wait_event(kpmap_ready)
            self.rplan = self._rplan_fill(rs, sizes)
            rfill_done = t.cuda.Event()
            rfill_done.record(main)
            self._mark("render fill queued")
        if pc is not None:
            with t.cuda.stream(side):
                sizes = pc["sizes"].get()  # waits for the side stream's copy only
                self._mark("adjust sizes read")
                if rfill_done is not None and os.environ.get("FVR_FILL_SERIAL", "0") == "1":
                    side.wait_event(rfill_done)
                self.plan = self._plan_fill(pc, sizes, side, keep)
                self.sample_plan = self.plan and self.sample_plan
                adjust_done = t.cuda.Event()
                adjust_done.record(side)
            # buffers from the side stream's pool that the loop's stream uses
            for buf in (getattr(self, "plan_entries", None), getattr(self, "plan_entries_b", None),
                        getattr(self, "plan_slice_len", None), getattr(self, "plan_slice_off", None),
                        getattr(self, "plan_row_of_pos", None), getattr(self, "sample_meta", None),
                        getattr(self, "rho", None)):
                if buf is not None:
                    buf.record_stream(main)
            main.wait_event(adjust_done)
        del keep
        self._mark("adjust fill queued")
        if self.layout_kind and not self.rplan:
            # float4 per (key point, channel), channels interleaved (fvr_stencil.cuh)
            self.layout = t.empty(shape + (C, 4), dtype=t.float32, device=dev)
            _lib.call("fvr_pack_layout", self.values.data_ptr(), C, self.grid, self.layout_kind,
                      self.layout.data_ptr(), _lib.stream_ptr())
        # work buffers (allocated once the plan builds are queued)
        self.residual = t.zeros((max(len(local), 1), self.h_bb, self.w_bb, self.pitch), dtype=t.float32,
                                device=dev)
        self.n_sq = V * self.bpv
        # [packed correction (C, n_kp) | sq partials (C, V*bpv) | vol partials (C, n_vol)] in one i64 buffer
        nvb = ctypes.c_int32(0)
        _lib.call("fvr_loop_volume_sq", None, None, None, self.n_kp, None, ctypes.byref(nvb), None, None)
        self.n_vol = int(nvb.value) if ground_truth is not None else 0
        a, b = C * self.n_kp, C * (self.n_kp + self.n_sq)
        self.comm = t.zeros(C * (self.n_kp + self.n_sq + self.n_vol) + 1, dtype=t.int64, device=dev)
        self.packed = self.comm[:a].view(C, self.n_kp)
        self.sq = self.comm[a:b].view(t.float64).view(C, self.n_sq)
        self.vol = self.comm[b:b + C * self.n_vol].view(t.float64).view(C, self.n_vol) if self.n_vol else None
        self.truth = None
        if ground_truth is not None:
            gt = np.ascontiguousarray(ground_truth, dtype=np.float32).reshape((C,) + shape)
            self.truth = t.from_numpy(gt).to(dev)
        self.state = t.zeros((C, 8), dtype=t.int32, device=dev)  # fvr_loop_state_t (32 B) per channel
        self.trace = t.zeros((C, max(self.max_iters, 1)), dtype=t.float64, device=dev)
        self.trace_vol = t.zeros((C, max(self.max_iters, 1)), dtype=t.float64, device=dev) \
            if ground_truth is not None else None
        self._mark("plans")
        if not self.plan:
            self.accum = t.zeros((C,) + shape, dtype=t.int64, device=dev)
        # A CUDA graph only pays off when an iteration is launch-bound (a few
        # tens of microseconds of device work); for larger problems the host
        # enqueues 3-4 launches (~30 us) far ahead of the device, and graph
        # instantiation costs milliseconds per call.
        small = V * self.w_bb * self.h_bb <= 65536
        self.use_graph = (use_graph and small and not self.sharded
                          and os.environ.get("FVR_NO_GRAPH") != "1") or os.environ.get("FVR_GRAPH") == "1"
        self.graph = None
        self.launches_per_iter = 0

    def _mark(self, name: str) -> None:
        if self._marks is not None:
            ev = self.t.cuda.Event(enable_timing=True)
            ev.record()
            self._marks.append((name, time.perf_counter(), ev))

    def init_profile(self):
        """[(section, host ms, device ms)] between FVR_INIT_PROFILE marks."""
        self.t.cuda.synchronize()
        m = self._marks or []
        return [(b[0], 1e3 * (b[1] - a[1]), a[2].elapsed_time(b[2])) for a, b in zip(m, m[1:])]

    def _layout_channel(self, ch: int):
        """Address of channel ch's first float4 in the interleaved layout."""
        return None if self.layout is None else self.layout.data_ptr() + 16 * ch

    # -- one iteration ---------------------------------------------------------
    def _rplan_row_order(self, row_len, n_units: int, tx: int, ty: int):
        """Rows of each tile of tx x ty units (one view) sorted longest first
        and dealt to the tile's units in order, so the 32 rows of a unit have
        similar lengths (SELL-C-sigma with sigma = the tile's pixels; config
        2, 16x16-pixel tiles: padded slots / entries 1.118 -> 1.036).
        Returns (row_src, unit_len) with row_src[r] = the natural row whose
        pixel row r renders."""
        t = self.t
        dev = row_len.device
        ux = (self.w_bb + 7) // 8
        uy = self.bpv // ux
        tiles_x, tiles_y = (ux + tx - 1) // tx, (uy + ty - 1) // ty
        unit = t.arange(n_units, device=dev)
        view, u = unit // self.bpv, unit % self.bpv
        tile = (view * tiles_y + (u // ux) // ty) * tiles_x + (u % ux) // tx
        tile_row = tile.repeat_interleave(32).long()
        r = t.arange(n_units * 32, device=dev)
        dest = t.argsort(tile_row * (n_units * 32) + r)
        src = t.argsort(tile_row * (1 << 20) + ((1 << 20) - 1 - row_len.long()))
        row_src = t.empty(n_units * 32, dtype=t.int32, device=dev)
        row_src[dest] = src.to(t.int32)
        unit_len = row_len[row_src.long()].view(n_units, 32).amax(1).to(t.int32).contiguous()
        return row_src, unit_len

    def _kp_map(self):
        """Lattice index -> index in the key-point list (-1 elsewhere)."""
        if getattr(self, "_kpmap", None) is None:
            t = self.t
            n_vox = int(np.prod(self.shape))
            self._kpmap = t.empty((n_vox,), dtype=t.int32, device=self.dev)
            _lib.call("fvr_kp_map", self.kp.data_ptr(), self.n_kp, n_vox, self._kpmap.data_ptr(), _lib.stream_ptr())
        return self._kpmap

    def _rplan_geo(self):
        return (self.cams.data_ptr(), self.v_end - self.v_begin, self.bbox.u0, self.bbox.v0, self.w_bb, self.h_bb,
                self.grid, self.params, _lib.ptr(self.occ), self.kp_dev.data_ptr())

    def _rplan_count(self):
        """Count pass of the render plan (enqueued only): (unit_len, row_len)."""
        if self.v_end <= self.v_begin:
            return None
        t = self.t
        n_units = (self.v_end - self.v_begin) * self.bpv
        unit_len = t.zeros(n_units, dtype=t.int32, device=self.dev)
        row_len = t.empty(n_units * 32, dtype=t.int32, device=self.dev) \
            if os.environ.get("FVR_RPLAN_TILE", "2x4") != "0" else None
        _lib.call("fvr_rplan_count", *self._rplan_geo(), unit_len.data_ptr(), _lib.ptr(row_len), _lib.stream_ptr())
        # the fill's static-positive stencil masks, computed now (off the fill's critical path)
        self._pos27 = None
        if not self._static_zero:
            self._pos27 = t.empty(int(np.prod(self.shape)), dtype=t.int32, device=self.dev)
            _lib.call("fvr_rplan_pos27", self.grid, self.kp_dev.data_ptr(), self.values.data_ptr(), self.nch,
                      self._pos27.data_ptr(), _lib.stream_ptr())
        return unit_len, row_len

    def _rplan_scan(self, unit_len, row_len) -> dict:
        """Row order and unit offsets of the render plan after its count pass
        (enqueued only; the total is read by _rplan_fill)."""
        t = self.t
        n_units = unit_len.numel()
        row_src = None
        al = int(_lib.load().fvr_rplan_chunk_entries())  # whole lane chunks of entries (fvr_rplan.cuh)
        tx, ty = (int(x) for x in os.environ.get("FVR_RPLAN_TILE", "2x4").split("x")) if row_len is not None \
            else (0, 0)
        buckets = int(os.environ.get("FVR_RPLAN_BUCKETS", "24"))
        if row_len is not None and (32 * tx * ty) & (32 * tx * ty - 1) == 0 and 32 * tx * ty <= 1024 \
                and buckets > 0 and os.environ.get("FVR_RPLAN_SORT", "1") == "1":
            # the whole layout in one native call (fvr_layout.cu)
            row_src = t.empty(n_units * 32, dtype=t.int32, device=self.dev)
            unit_len = t.empty(n_units, dtype=t.int32, device=self.dev)
            off = t.empty(n_units + 1, dtype=t.int64, device=self.dev)
            order = t.empty(n_units, dtype=t.int32, device=self.dev)
            totals = t.empty(2, dtype=t.int64, device=self.dev)
            _lib.call("fvr_rplan_layout", row_len.data_ptr(), self.v_end - self.v_begin, self.w_bb, self.h_bb, tx, ty,
                      al, buckets, row_src.data_ptr(), unit_len.data_ptr(), off.data_ptr(), order.data_ptr(),
                      totals.data_ptr(), _lib.stream_ptr())
            return dict(unit_len=unit_len, row_src=row_src, off=off, order=order, sizes=totals)
        if row_len is not None:
            if (32 * tx * ty) & (32 * tx * ty - 1) == 0 and 32 * tx * ty <= 1024:  # one kernel per call
                row_src = t.empty(n_units * 32, dtype=t.int32, device=self.dev)
                unit_len = t.empty(n_units, dtype=t.int32, device=self.dev)
                _lib.call("fvr_rplan_tile_rows", row_len.data_ptr(), self.v_end - self.v_begin, self.w_bb, self.h_bb,
                          tx, ty, al, row_src.data_ptr(), unit_len.data_ptr(), _lib.stream_ptr())
            else:
                row_src, unit_len = self._rplan_row_order(row_len, n_units, tx, ty)
        unit_len = (unit_len + al - 1) & ~(al - 1)
        off = t.zeros(n_units + 1, dtype=t.int64, device=self.dev)
        off[1:] = t.cumsum(unit_len.long(), 0)
        mx = unit_len.max()
        # fill and render visit the units longest first (a short tail); the
        # order is computed before the sizes reach the host
        order = self._rplan_unit_order(unit_len, mx) if os.environ.get("FVR_RPLAN_SORT", "1") == "1" else None
        return dict(unit_len=unit_len, row_src=row_src, off=off, order=order, sizes=t.stack([off[-1], mx.long()]))

    def _rplan_unit_order(self, unit_len, max_len):
        """The order fill and render visit the units: longest first, in
        ``buckets`` length classes (a short tail), and inside a class by
        tiles of 2x4 units (16x16 pixels), so the 8 warps of a CTA render
        neighbouring pixels and share the operand in L1 (config 2:
        0.1244 ms sorted by length alone, 0.1188 ms bucketed and tiled)."""
        t = self.t
        n_units = unit_len.numel()
        buckets = int(os.environ.get("FVR_RPLAN_BUCKETS", "24"))
        if buckets <= 0:
            return t.argsort(unit_len, descending=True).to(t.int32)
        mx = max_len.to(t.int32).reshape(1)  # device scalar: no synchronisation
        keys = t.empty(n_units, dtype=t.int64, device=unit_len.device)
        _lib.call("fvr_rplan_unit_keys", unit_len.data_ptr(), self.v_end - self.v_begin, self.w_bb, self.h_bb,
                  buckets, mx.data_ptr(), keys.data_ptr(), _lib.stream_ptr())
        return t.sort(keys).indices.to(t.int32)

    def _rplan_fill(self, rs: dict, sizes) -> bool:
        """B of rec = B c + base + t_fin bg in SELL-32 form (fvr_rplan.cuh),
        filled on the current stream; False when it would not fit."""
        t = self.t
        dev = self.dev
        stream = _lib.stream_ptr()
        unit_len, off = rs["unit_len"], rs["off"]
        n_units = unit_len.numel()
        geo = self._rplan_geo()
        self.rp_row_src = rs["row_src"]
        slots = int(sizes[0]) * 32
        # 6-byte entries (24-bit column) unless the hull has >= 2^24 key
        # points (or FVR_WIDE_PLANS=1): then 8-byte (u32 column, f32 weight)
        self.rp_wide = self.n_kp >= (1 << 24) or os.environ.get("FVR_WIDE_PLANS") == "1"
        need = (8 if self.rp_wide else 6) * slots + 8 * (self.nch + 1) * n_units * 32
        if need > self.PLAN_MAX_BYTES:
            return False
        try:  # (no cudaMemGetInfo probe: it synchronises and costs tens of ms)
            # every chunk, padding included, is written by the fill (no clearing)
            ent_a = t.empty(max(slots, 2), dtype=t.int32, device=dev)
            ent_b = t.empty(max(slots if self.rp_wide else slots // 2, 1), dtype=t.int32, device=dev)
            # the fill writes every row's base and t_fin (overhanging rows too)
            base = t.empty((self.nch, n_units * 32), dtype=t.float64, device=dev)
            t_fin = t.empty(n_units * 32, dtype=t.float64, device=dev)
            # the operand: max(v, 0) per hull key point (float4 for 3 channels)
            kpv = t.empty((max(self.n_kp, 1),) + ((4,) if self.nch == 3 else ()), dtype=t.float32, device=dev)
        except t.cuda.OutOfMemoryError:
            return False
        self.rp_order = rs["order"]
        _lib.call("fvr_rplan_fill", *geo, None if self._static_zero else self.values.data_ptr(), self.nch,
                  off.data_ptr(), _lib.ptr(self.rp_order),
                  _lib.ptr(self.rp_row_src), self._kp_map().data_ptr(), ent_a.data_ptr(), ent_b.data_ptr(),
                  base.data_ptr(), t_fin.data_ptr(), _lib.ptr(getattr(self, "_pos27", None)), int(self.rp_wide),
                  stream)
        self._pos27 = None
        _lib.call("fvr_rplan_pack", self.values.data_ptr(), self.nch, self.grid, self.kp.data_ptr(), self.n_kp,
                  kpv.data_ptr(), None, stream)
        self.rp_len, self.rp_off, self.rp_base, self.rp_tfin = unit_len, off, base, t_fin
        self.rp_a, self.rp_b, self.rp_kpv = ent_a, ent_b, kpv
        self.rplan_nnz = slots
        return True

    def _render(self, stream):
        self._host_small = None  # (every iteration starts here: staged states / traces are stale)
        if self.v_end <= self.v_begin:
            return 0
        if self.rplan:
            n = 1
            if not self.plan:  # the scatter fallback's update does not maintain the operand
                _lib.call("fvr_rplan_pack", self.values.data_ptr(), self.nch, self.grid, self.kp.data_ptr(),
                          self.n_kp, self.rp_kpv.data_ptr(), self.state.data_ptr(), stream)
                n += 1
            _lib.call(
                "fvr_rplan_render", self.rp_len.data_ptr(), self.rp_off.data_ptr(), self.rp_a.data_ptr(),
                self.rp_b.data_ptr(),
                # the loop's own initial lattice has no static term (base is all zeros), and a zero
                # background needs no t_fin: neither is streamed then
                None if self._static_zero else self.rp_base.data_ptr(),
                self.rp_tfin.data_ptr() if any(b != 0.0 for b in self.background) else None,
                _lib.ptr(self.rp_order),
                _lib.ptr(self.rp_row_src), self.v_end - self.v_begin, self.w_bb, self.h_bb, self.src.data_ptr(),
                self.rp_kpv.data_ptr(), self.nch, self.background, self.residual.data_ptr(),
                self.sq[0, self.v_begin * self.bpv:].data_ptr(), self.n_sq, self.state.data_ptr(),
                self._fused_finalize(), int(self.rp_wide), stream,
            )
            return n
        _lib.call(
            "fvr_loop_render", self.cams.data_ptr(), self.v_end - self.v_begin, self.bbox.u0,
            self.bbox.v0, self.w_bb, self.h_bb, self.src.data_ptr(), self.values.data_ptr(),
            _lib.ptr(self.layout), _lib.ptr(self.occ), self.grid, self.params, self.background, self.nch,
            _lib.ptr(self.scat), self.residual.data_ptr(), self.sq[0, self.v_begin * self.bpv:].data_ptr(),
            self.n_sq, self.state.data_ptr(), stream,
        )
        return 1

    def _adjust(self, stream):
        if self.n_rays == 0:
            return 0
        c = self.cfg
        for ch in range(self.nch):
            _lib.call(
                "fvr_loop_adjust", self.cams.data_ptr(), self.rays.data_ptr(), self.n_rays,
                self.bbox.u0, self.bbox.v0, self.w_bb, self.h_bb, self.residual.data_ptr() + 4 * ch, self.pitch,
                self.inside.data_ptr(), self.grid, c.tau, c.alpha_l, c.alpha_d_eff,
                1 if c.stochastic else 0, c.g_sigma, c.seed & 0xFFFFFFFFFFFFFFFF, self.ray_base,
                self.accum[ch].data_ptr(), self.state[ch].data_ptr(), stream,
            )
        return self.nch

    def _volume(self, stream):
        if self.truth is None:
            return 0
        nvb = ctypes.c_int32(0)
        for ch in range(self.nch):
            _lib.call(
                "fvr_loop_volume_sq", self.values[ch].data_ptr(), self.truth[ch].data_ptr(), self.kp.data_ptr(),
                self.n_kp, self.vol[ch].data_ptr(), ctypes.byref(nvb), self.state[ch].data_ptr(), stream,
            )
        return self.nch

    def _fused(self) -> bool:
        """The render plan's last block runs finalize (single-rank loops with
        the gather adjust; the scatter fallback keeps the separate launch)."""
        return (self.rplan and self.plan and not self.sharded
                and os.environ.get("FVR_FUSED_FINALIZE", "1") == "1")

    def _fused_finalize(self):
        if not self._fused():
            return None
        if getattr(self, "_fin_args", None) is None:
            f = _lib.FvrLoopFinalize()
            f.n_views = self.n_views
            f.blocks_per_view = self.bpv
            f.pixels_per_view = self.w_bb * self.h_bb
            f.vol_partials = _lib.ptr(self.vol)
            f.n_vol_blocks = self.n_vol
            f.n_kp = self.n_kp
            f.converge_eps = self.cfg.converge_eps
            f.trace_rmse = self.trace.data_ptr()
            f.trace_vol = _lib.ptr(self.trace_vol)
            f.trace_stride = self.trace.shape[1]
            # per-view fixed-point sums the render's units accumulate (+ an overflow flag per channel)
            self._sq_acc = self.t.zeros(self.nch * (self.n_views + 1), dtype=self.t.int64, device=self.dev)
            f.sq_accum = self._sq_acc.data_ptr()
            if self.sample_plan and self.rho is not None and os.environ.get("FVR_L2_DISCARD", "1") == "1":
                # rho is dead between the gather and the next weigh pass: drop its dirty L2 lines
                f.l2_discard = self.rho.data_ptr()
                f.l2_discard_bytes = self.rho.numel() * self.rho.element_size()
            self._fin_args = f
        return ctypes.addressof(self._fin_args)

    def _finalize(self, stream):
        pix = self.w_bb * self.h_bb
        for ch in range(self.nch):
            _lib.call(
                "fvr_loop_finalize", self.sq[ch].data_ptr(), self.n_views, self.bpv, pix,
                _lib.ptr(None if self.vol is None else self.vol[ch]), self.n_vol, self.n_kp, self.cfg.converge_eps,
                self.trace[ch].data_ptr(), _lib.ptr(None if self.trace_vol is None else self.trace_vol[ch]),
                self.state[ch].data_ptr(), stream,
            )
        return self.nch

    def _update(self, stream):
        if self.n_kp == 0:
            return 0
        for ch in range(self.nch):
            _lib.call(
                "fvr_loop_update", self.values[ch].data_ptr(), self.accum[ch].data_ptr(), self.kp.data_ptr(),
                self.n_kp, self._layout_channel(ch), self.layout_kind, self.nch, self.grid,
                self.state[ch].data_ptr(), stream,
            )
        return self.nch

    def _allreduce(self, stream):
        """Sum corrections and RMSE partials over ranks (exact: int64)."""
        for ch in range(self.nch if self.n_kp else 0):
            _lib.call("fvr_pack_correction", self.accum[ch].data_ptr(), self.kp.data_ptr(), self.n_kp,
                      self.packed[ch].data_ptr(), stream)
        exchange(self.comm, self.sq, self.vol, self.v_begin, self.v_end, self.bpv, self.rank, stream=stream)
        for ch in range(self.nch if self.n_kp else 0):
            _lib.call("fvr_unpack_correction", self.packed[ch].data_ptr(), self.kp.data_ptr(), self.n_kp,
                      self.accum[ch].data_ptr(), stream)
        return 2 * self.nch if self.n_kp else 0

    # -- the back-projection plan (deterministic mode) --------------------------
    # plans larger than this (or that do not fit) fall back to the kernels they replace
    PLAN_MAX_BYTES = 48 << 30

    def _plan_count(self) -> dict:
        """Count pass and SELL layout of the back-projection operator
        (fvr_plan.cu): row = hull key point, entry = (residual pixel, W)
        merged per ray run in deterministic mode, (in-hull sample id, W)
        unmerged in stochastic mode.  Enqueued only: the sizes are read by
        _plan_fill together with the render plan's (one synchronisation)."""
        t = self.t
        dev = self.dev
        stream = _lib.stream_ptr()
        # deterministic entries are 6 bytes (24-bit residual index) unless V * P
        # >= 2^24 (or FVR_WIDE_PLANS=1): then int2 (residual index, f32 W)
        self.adj_wide = not self.sample_plan and (
            (self.v_end - self.v_begin) * self.w_bb * self.h_bb >= (1 << 24) or os.environ.get("FVR_WIDE_PLANS") == "1")
        kp_map = self._kp_map()
        counts = t.zeros(self.n_kp, dtype=t.int32, device=dev)
        geo = (self.cams.data_ptr(), self.rays.data_ptr(), self.n_rays, self.bbox.u0, self.bbox.v0, self.w_bb,
               self.h_bb, self.inside.data_ptr(), self.grid)
        ray_samples = None
        if self.sample_plan:
            ray_samples = t.zeros(self.n_rays, dtype=t.int32, device=dev)
            _lib.call("fvr_sample_plan_count", *geo, kp_map.data_ptr(), counts.data_ptr(), ray_samples.data_ptr(),
                      stream)
        else:
            _lib.call("fvr_adjust_plan_count", *geo, kp_map.data_ptr(), counts.data_ptr(), stream)
        # SELL-32 layout: slices of 32 rows; FVR_SELL_SORT=1 sorts rows longest
        # first (least padding), else key-point order (neighbouring rows share
        # rays, so their residual / rho reads share cache lines) sorted by
        # length within windows of sigma rows (SELL-C-sigma; config 2:
        # sigma 0 / 64 / 128 / 512 / 4096: 0.0783 / 0.0773 / 0.0760 / 0.0767 /
        # 0.0844 ms; with the final pipelined gather 32 / 64 / 128 / 256:
        # 0.0501 / 0.0488 / 0.0486 / 0.0519 ms, and the sample plan's gather
        # 0.0978 / 0.0969 / 0.0985 / 0.1025 ms -- so 64 for the sample plan)
        sigma = int(os.environ.get("FVR_SELL_SIGMA", "64" if self.sample_plan else "128"))
        # whole lane chunks (fvr_plan.cu): 16 bytes of six-byte entries (8), or
        # 32 bytes of eight-byte (wide) entries (kSE = 4); the sample plan's
        # format is decided after the sizes reach the host, so it pads to 8
        pad = 4 if self.adj_wide else 8
        if os.environ.get("FVR_SELL_SORT", "0") != "1" and 2 <= sigma <= 1024 and sigma & (sigma - 1) == 0:
            # the whole layout in one native call (fvr_layout.cu)
            n_slices = (self.n_kp + 31) // 32
            row_of_pos = t.empty(self.n_kp, dtype=t.int32, device=dev)
            slice_len = t.empty(n_slices, dtype=t.int32, device=dev)
            slice_off = t.empty(n_slices + 1, dtype=t.int64, device=dev)
            row_info = t.empty(self.n_kp, dtype=t.int64, device=dev)
            totals = t.empty(3, dtype=t.int64, device=dev)
            sid0 = t.empty(self.n_rays, dtype=t.int64, device=dev) if ray_samples is not None else None
            _lib.call("fvr_sell_layout", counts.data_ptr(), self.n_kp, sigma, pad, _lib.ptr(ray_samples), self.n_rays,
                      _lib.ptr(sid0), row_of_pos.data_ptr(), slice_len.data_ptr(), slice_off.data_ptr(),
                      row_info.data_ptr(), totals.data_ptr(), stream)
            return dict(geo=geo, kp_map=kp_map, ray_samples=ray_samples, sid0=sid0, row_of_pos=row_of_pos,
                        slice_len=slice_len, slice_off=slice_off, row_info=row_info, sizes=totals)
        if os.environ.get("FVR_SELL_SORT", "0") == "1":
            order = t.argsort(counts, descending=True)
        elif 2 <= sigma <= 1024 and sigma & (sigma - 1) == 0:  # one kernel: bitonic per window
            order = t.empty(self.n_kp, dtype=t.int32, device=dev)
            _lib.call("fvr_sell_window_order", counts.data_ptr(), self.n_kp, sigma, order.data_ptr(), stream)
        elif sigma > 0:  # sorted within windows of sigma neighbouring rows
            pos = t.arange(self.n_kp, device=dev)
            order = t.argsort((pos // sigma) * (1 << 24) + ((1 << 24) - 1 - counts.long()))
        else:
            order = t.arange(self.n_kp, device=dev)
        row_of_pos = order.to(t.int32)
        row_pos = t.empty_like(row_of_pos)
        row_pos[order.long()] = t.arange(self.n_kp, dtype=t.int32, device=dev)
        n_slices = (self.n_kp + 31) // 32
        slice_len = t.zeros(n_slices * 32, dtype=t.int32, device=dev)
        slice_len[: self.n_kp] = counts[order]
        slice_len = slice_len.view(n_slices, 32).amax(1).contiguous()
        slice_len = (slice_len + pad - 1) & ~(pad - 1)
        slice_off = t.zeros(n_slices + 1, dtype=t.int64, device=dev)
        slice_off[1:] = t.cumsum(slice_len.long(), 0)
        sizes = [slice_off[-1], counts.long().sum()]
        sizes.append(ray_samples.long().sum() if ray_samples is not None else sizes[1] * 0)
        # each row's SELL position in one word: slice entry offset << 5 | lane
        rp = row_pos.long()
        row_info = (slice_off[rp >> 5] << 5) | (rp & 31)
        return dict(geo=geo, kp_map=kp_map, ray_samples=ray_samples, row_of_pos=row_of_pos, slice_len=slice_len,
                    slice_off=slice_off, row_info=row_info, sizes=t.stack(sizes))

    def _plan_fill(self, pc: dict, sizes, stream, keep: list) -> bool:
        """Allocate, clear and fill the plan on ``stream`` (the current
        stream); the temporaries the fill reads go to ``keep`` until it is
        done.  False (scatter fallback) when the plan would not fit."""
        t = self.t
        dev = self.dev
        c = self.cfg
        slots = int(sizes[0]) * 32
        nnz = int(sizes[1])
        n_samples = int(sizes[2]) if self.sample_plan else 0
        # the sample plan's entries are 6 bytes while sample ids fit 24 bits
        self.splan_e6 = self.sample_plan and n_samples < (1 << 24) and os.environ.get("FVR_WIDE_PLANS") != "1"
        # entries + per-sample (meta: 8 B, rho: 4 B per channel slot) + the cursor
        need = (8 if ((self.sample_plan and not self.splan_e6) or self.adj_wide) else 6) * slots + \
            (2 + 4 * self.pitch) * n_samples + 8 * self.n_kp
        if need > self.PLAN_MAX_BYTES or n_samples >= 2 ** 31:
            return False
        pad_zero = os.environ.get("FVR_PAD_ZERO", "1") == "1"
        try:
            cursor = t.zeros(self.n_kp, dtype=t.int64, device=dev)
            if (self.sample_plan and not self.splan_e6) or self.adj_wide:  # int2 (sample id / residual index, W)
                entries = t.zeros(max(2 * slots, 2), dtype=t.int32, device=dev)
                entries_b = None
            else:  # 6 bytes: sample id or residual index (24 bits) + 24-bit weight
                # (the padding is cleared after the fill from its final cursors:
                # no full-buffer clear on the side stream ahead of the fill)
                alloc = t.empty if pad_zero else t.zeros
                entries = alloc(max(slots, 2), dtype=t.int32, device=dev)
                entries_b = alloc(max(slots // 2, 1), dtype=t.int32, device=dev)
            if self.sample_plan:
                meta = t.empty(max(n_samples // 2, 2), dtype=t.int32, device=dev)  # int2 per 4-slot block
                rho = t.zeros((max(n_samples, 1), self.pitch), dtype=t.float32, device=dev)
        except t.cuda.OutOfMemoryError:
            return False
        sell = (pc["row_info"].data_ptr(), cursor.data_ptr(), entries.data_ptr())
        keep += [pc, cursor]
        stream = stream.cuda_stream
        if self.sample_plan:
            sid0 = pc.get("sid0")
            if sid0 is None:  # (the non-native SELL layout variants)
                sid0 = t.zeros(self.n_rays, dtype=t.int64, device=dev)
                sid0[1:] = t.cumsum(pc["ray_samples"][:-1].long(), 0)
            self.rho = rho
            keep.append(sid0)
            n_blocks = n_samples // 4
            # renumber the blocks spatially (Morton order of each group's first
            # cell) so a slice's rho reads sit close together
            spatial = max(self.shape) <= 1024 and os.environ.get("FVR_SPLAN_SPATIAL", "1") == "1" and n_blocks > 0
            keys = t.empty(n_blocks, dtype=t.int64, device=dev) if spatial else None
            _lib.call("fvr_sample_plan_fill", *pc["geo"], c.tau, c.alpha_l, c.alpha_d_eff,
                      pc["kp_map"].data_ptr(), sid0.data_ptr(), *sell, _lib.ptr(entries_b), meta.data_ptr(),
                      _lib.ptr(keys), stream)
            if pad_zero and entries_b is not None:  # before the renumbering reads every slot
                self._pad_zero(pc, cursor, entries, entries_b, stream)
            if spatial:
                meta_new = t.empty_like(meta)
                _lib.call("fvr_sample_plan_spatial", entries.data_ptr(), slots, int(entries_b is not None),
                          keys.data_ptr(), n_blocks, meta.data_ptr(), meta_new.data_ptr(), stream)
                meta = meta_new
            if entries_b is not None and os.environ.get("FVR_SPLAN_SORT", "0") == "1":
                # each row by sample id: a warp's lanes then read nearby rho lines together
                _lib.call("fvr_plan_sort_rows", pc["slice_len"].data_ptr(), pc["slice_off"].data_ptr(),
                          pc["slice_len"].numel(), entries.data_ptr(), entries_b.data_ptr(), stream)
            self.sample_meta = meta
            self.n_samples = n_samples
        else:
            _lib.call("fvr_adjust_plan_fill", *pc["geo"], c.tau, c.alpha_l, c.alpha_d_eff,
                      pc["kp_map"].data_ptr(), *sell, _lib.ptr(entries_b), stream)
            if pad_zero and entries_b is not None:
                self._pad_zero(pc, cursor, entries, entries_b, stream)
        self.plan_slice_len = pc["slice_len"]
        self.plan_slice_off = pc["slice_off"]
        self.plan_row_of_pos = pc["row_of_pos"]
        self.plan_entries = entries
        self.plan_entries_b = entries_b
        self.plan_nnz = nnz
        self.plan_slots = slots
        return True

    def _pad_zero(self, pc, cursor, entries, entries_b, stream):
        _lib.call("fvr_sell_pad_zero", cursor.data_ptr(), pc["row_of_pos"].data_ptr(), self.n_kp,
                  pc["slice_len"].data_ptr(), pc["slice_off"].data_ptr(), pc["slice_len"].numel(),
                  entries.data_ptr(), entries_b.data_ptr(), stream)

    def _weigh(self, stream):
        """rho = residual * G per in-hull sample (stochastic sample plan)."""
        c = self.cfg
        _lib.call("fvr_loop_weighted_residual", self.sample_meta.data_ptr(), self.n_samples,
                  self.rays.data_ptr(), self.w_bb, self.h_bb, self.residual.data_ptr(), self.nch,
                  c.seed & 0xFFFFFFFFFFFFFFFF, c.g_sigma, self.ray_base, self.rho.data_ptr(),
                  self.state.data_ptr(), 1 if self._fused() else 0, stream)
        return 1

    def _gather(self, stream, packed: bool):
        if self.n_kp == 0:
            return 0
        src = self.rho if self.sample_plan else self.residual
        _lib.call("fvr_loop_gather", self.plan_slice_len.data_ptr(), self.plan_slice_off.data_ptr(),
                  self.plan_row_of_pos.data_ptr(), self.plan_entries.data_ptr(), _lib.ptr(self.plan_entries_b),
                  self.n_kp,
                  src.data_ptr(), self.nch, self.kp.data_ptr(), self.values.data_ptr(),
                  _lib.ptr(self.layout), self.layout_kind, self.grid,
                  _lib.ptr(self.rp_kpv) if self.rplan else None, self.packed.data_ptr() if packed else None,
                  self.state.data_ptr(), int(self.sample_plan), stream)
        return 1

    def _update_packed(self, stream):
        if self.n_kp == 0:
            return 0
        for ch in range(self.nch):
            kpv = self.rp_kpv.data_ptr() + 4 * ch if self.rplan else None
            _lib.call("fvr_loop_update_packed", self.packed[ch].data_ptr(), self.n_kp, self.kp.data_ptr(),
                      self.values[ch].data_ptr(), self._layout_channel(ch), self.layout_kind, self.nch, self.grid,
                      kpv, 1 if self.nch == 1 else 4, self.state[ch].data_ptr(), stream)
        return self.nch

    def _allreduce_packed(self, stream):
        """All-reduce [packed | sq | vol] once the gather filled ``packed``."""
        exchange(self.comm, self.sq, self.vol, self.v_begin, self.v_end, self.bpv, self.rank, stream=stream)
        return 0

    def stages(self):
        """[(name, fn(stream) -> launches)] of one iteration, in order; the
        name 'decision' marks where the convergence rule has been evaluated."""
        vol = [("volume", self._volume)] if self.truth is not None else []  # vol_rmse partials
        if self._fused():  # render -> finalize in one launch; the volume partials first
            s = vol + [("render", self._render)]
            if self.sample_plan:
                s += [("weigh", self._weigh)]
            return s + [("decision", None), ("adjust", lambda st: self._gather(st, False))]
        s = [("render", self._render)] + vol
        if self.sample_plan:
            s += [("weigh", self._weigh)]
        if self.plan:
            if self.sharded:
                s += [("adjust", lambda st: self._gather(st, True)), ("allreduce", self._allreduce_packed),
                      ("finalize", self._finalize), ("decision", None), ("update", self._update_packed)]
            else:
                s += [("finalize", self._finalize), ("decision", None),
                      ("adjust", lambda st: self._gather(st, False))]
        else:
            s += [("adjust", self._adjust)]
            if self.sharded:
                s += [("allreduce", self._allreduce)]
            s += [("finalize", self._finalize), ("decision", None), ("update", self._update)]
        return s

    def pre_decision(self, stream) -> int:
        n = 0
        for name, fn in self.stages():
            if name == "decision":
                break
            n += fn(stream)
        return n

    def post_decision(self, stream) -> int:
        n, after = 0, False
        for name, fn in self.stages():
            if after:
                n += fn(stream)
            after = after or name == "decision"
        return n

    def launch_iteration(self) -> None:
        stream = _lib.stream_ptr()
        self.launches_per_iter = self.pre_decision(stream) + self.post_decision(stream)

    def capture(self) -> None:
        """Capture one iteration into a CUDA graph (single-GPU only)."""
        # capture_begin/end directly: the torch.cuda.graph context manager also
        # runs gc.collect() and empty_cache(), which cost 2-300 ms per call
        t = self.t
        g = t.cuda.CUDAGraph()
        side = t.cuda.Stream()
        side.wait_stream(t.cuda.current_stream())
        with t.cuda.stream(side):
            g.capture_begin(capture_error_mode="thread_local")
            try:
                self.launch_iteration()
            finally:
                g.capture_end()
        t.cuda.current_stream().wait_stream(side)
        self.graph = g

    def step(self) -> None:
        self._host_values = self._host_small = None  # staged result copies are stale once the loop moves
        if self.graph is not None:
            self.graph.replay()
        else:
            self.launch_iteration()

    # -- the loop ----------------------------------------------------------------
    def reset_state(self) -> None:
        self._host_small = None
        self.state.zero_()
        if self.accum is not None:
            self.accum.zero_()

    def read_states(self) -> list[dict]:
        small = getattr(self, "_host_small", None)
        states = small[0] if small is not None else self.state.cpu().numpy()
        out = []
        for s in states:
            prev = s[4:6].copy().view(np.float64)[0]
            out.append({"it": int(s[0]), "done": int(s[1]), "converged": int(s[2]), "prev_rmse": float(prev)})
        return out

    def read_state(self) -> dict:
        """Channel 0's state (the only one of a single-channel loop)."""
        return self.read_states()[0]

    def run(self, callback=None, chunk: int = 8, snapshot=None):
        """Iterate until the rule fires (in every channel) or max_iters;
        returns (iterations, converged, wall_ms per iteration) of channel 0 --
        read_states() has every channel's.  ``callback(channel, it, values,
        rmse)`` fires after every iteration's RMSE with a host copy of that
        channel's lattice (see _run_with_snapshots)."""
        t = self.t
        if callback is not None:
            return self._run_with_snapshots(callback, snapshot=snapshot)
        if self.use_graph and self.graph is None and self.max_iters > 1:
            self.capture()
        # keep one chunk in flight: after enqueueing chunk i, wait for chunk
        # i-1's state copy and stop once every channel's sticky `done` is set
        bufs = [t.zeros((self.nch, 8), dtype=t.int32, pin_memory=True) for _ in range(2)]
        events = [None, None]
        issued, i = 0, 0
        t_start = time.perf_counter()
        while issued < self.max_iters:
            n = min(chunk, self.max_iters - issued)
            for _ in range(n):
                self.step()
            issued += n
            b = i & 1
            bufs[b].copy_(self.state, non_blocking=True)
            events[b] = t.cuda.Event()
            events[b].record()
            if i >= 1:
                events[b ^ 1].synchronize()
                if bool(bufs[b ^ 1][:, 1].all()):
                    break
            i += 1
        self._stage_values()
        t.cuda.synchronize()
        self.total_ms = (time.perf_counter() - t_start) * 1e3
        st = self.read_state()
        it = st["it"]
        wall = [self.total_ms / max(it, 1)] * it
        return it, bool(st["converged"]), wall

    def _run_with_snapshots(self, callback, depth: int = 3, snapshot=None):
        """The loop with per-iteration snapshots that do not stall it (§8f rank 4).

        After an iteration's RMSE, the lattice and the loop state are copied
        device-to-device into one of ``depth`` ring slots on the loop's stream
        (before the update can change them); a side stream moves the slot to
        page-locked host memory while the device runs the next iterations.
        The host delivers snapshots in iteration order, at the latest when a
        slot is about to be reused, so at most ``depth`` iterations run ahead
        of the callbacks.  Iterations issued after the rule fired are no-ops
        (sticky ``done``) and deliver nothing.

        ``snapshot`` (optional) replaces the lattice copy by a device-side
        transform: ``snapshot.shape`` is the per-slot f32 buffer shape,
        ``snapshot.init(buf)`` prepares a slot's device buffer once and
        ``snapshot.fill(values, buf, stream)`` fills it from the lattice on the
        loop's stream; the callback then receives the host copy of ``buf``
        (reconstruct_temperature: green -> T -> RGB in one launch)."""
        t = self.t
        C = self.nch
        main = t.cuda.current_stream()
        side = t.cuda.Stream()
        stream = _lib.stream_ptr()
        shape = tuple(self.values.shape) if snapshot is None else tuple(snapshot.shape)
        host = _pinned_ring(shape, t.float32, depth)
        host_st = _pinned_ring(tuple(self.state.shape), t.int32, depth)
        slots = [{"dev": t.empty(shape, dtype=t.float32, device=self.dev), "st_dev": t.empty_like(self.state),
                  "host": host[i], "st": host_st[i], "ev": None} for i in range(depth)]
        if snapshot is not None:
            for s in slots:
                snapshot.init(s["dev"])
        delivered = [0] * C

        def deliver(slot) -> bool:
            slot["ev"].synchronize()
            slot["ev"] = None
            st = slot["st"].numpy()
            all_done = True
            for c in range(C):
                it_c = int(st[c, 0])
                if it_c > delivered[c]:
                    rmse = float(st[c, 4:6].copy().view(np.float64)[0])
                    callback(c, it_c, (slot["host"][c] if snapshot is None else slot["host"]).numpy().copy(), rmse)
                    delivered[c] = it_c
                all_done = all_done and bool(st[c, 1])
            return all_done

        t_start = time.perf_counter()
        issued = k = 0
        finished = False
        while issued < self.max_iters and not finished:
            slot = slots[k % depth]
            if slot["ev"] is not None and deliver(slot):
                finished = True
                break
            self.pre_decision(stream)
            if snapshot is None:
                slot["dev"].copy_(self.values)
            else:
                snapshot.fill(self.values, slot["dev"], stream)
            slot["st_dev"].copy_(self.state)
            ready = t.cuda.Event()
            ready.record(main)
            side.wait_event(ready)
            with t.cuda.stream(side):
                slot["host"].copy_(slot["dev"], non_blocking=True)
                slot["st"].copy_(slot["st_dev"], non_blocking=True)
                slot["ev"] = t.cuda.Event()
                slot["ev"].record(side)
            self.post_decision(stream)
            issued += 1
            k += 1
        for j in range(depth):  # drain the ring in iteration order
            slot = slots[(k + j) % depth]
            if slot["ev"] is not None:
                deliver(slot)
        self._stage_values()
        t.cuda.synchronize()
        self.total_ms = (time.perf_counter() - t_start) * 1e3
        st = self.read_state()
        it = st["it"]
        return it, bool(st["converged"]), [self.total_ms / max(it, 1)] * it

    # -- results -----------------------------------------------------------------
    def _stage_values(self) -> None:
        """Queue the lattice's D2H into page-locked memory behind the last
        iteration; the pinned allocation overlaps the device work still in
        flight (a pageable .cpu() of 8.6 MB at 128^3 costs about 3 ms).  The
        loop states and traces ride along, so reading them after the run
        costs no further round trip."""
        t = self.t
        host = t.empty(tuple(self.values.shape), dtype=t.float32, pin_memory=True)
        host.copy_(self.values, non_blocking=True)
        self._host_values = host
        st = t.empty(tuple(self.state.shape), dtype=self.state.dtype, pin_memory=True)
        st.copy_(self.state, non_blocking=True)
        tr = t.empty(tuple(self.trace.shape), dtype=self.trace.dtype, pin_memory=True)
        tr.copy_(self.trace, non_blocking=True)
        tv = None
        if self.trace_vol is not None:
            tv = t.empty(tuple(self.trace_vol.shape), dtype=self.trace_vol.dtype, pin_memory=True)
            tv.copy_(self.trace_vol, non_blocking=True)
        self._host_small = (st.numpy(), tr.numpy(), None if tv is None else tv.numpy())

    def host_values(self) -> np.ndarray:
        host, self._host_values = getattr(self, "_host_values", None), None
        if host is not None:
            self.t.cuda.current_stream().synchronize()
            v = host.numpy()  # keeps the pinned tensor alive
        else:
            v = self.values.cpu().numpy()
        return v[0] if self.nch == 1 else v

    def host_trace(self, iterations: int, channel: int = 0):
        small = getattr(self, "_host_small", None)
        if small is not None:  # staged with the lattice after run()
            rmse = small[1][channel, :iterations].tolist()
            vol = small[2][channel, :iterations].tolist() if small[2] is not None else []
            return rmse, vol
        rmse = self.trace[channel, :iterations].cpu().numpy().tolist()
        vol = self.trace_vol[channel, :iterations].cpu().numpy().tolist() if self.trace_vol is not None else []
        return rmse, vol
