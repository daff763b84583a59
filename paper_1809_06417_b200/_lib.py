"""ctypes binding of ``libfvr_b200.so`` (the C ABI in ``include/fvr_b200.h``).

The library is built in-tree (``__graft_entry__.build()`` or ``make -C
paper_1809_06417_b200/csrc``).  There is no CPU fallback: when the library or
a CUDA device is missing, every compute entry point raises ``RuntimeError``.
Device memory is owned by torch tensors; only raw pointers and the current
CUDA stream cross the boundary.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_int, c_int32, c_int64, c_uint64, c_void_p

from .errors import EmptyHullError, NoFlameError

# FVR_LIB selects an experiment build of the same library (csrc/Makefile OUT=...)
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), os.environ.get("FVR_LIB", "libfvr_b200.so"))

FVR_OK = 0
FVR_ERR_INVALID = 1
FVR_ERR_CUDA = 2
FVR_ERR_EMPTY_HULL = 3
FVR_ERR_NO_FLAME = 4


class FvrGrid(ctypes.Structure):
    _fields_ = [
        ("nx", c_int32),
        ("ny", c_int32),
        ("nz", c_int32),
        ("reserved", c_int32),
        ("origin", c_double * 3),
        ("edge", c_double),
    ]


class FvrCamera(ctypes.Structure):
    _fields_ = [
        ("fx", c_double),
        ("fy", c_double),
        ("cx", c_double),
        ("cy", c_double),
        ("rotation", c_double * 9),
        ("center", c_double * 3),
        ("width", c_int32),
        ("height", c_int32),
    ]


class FvrRenderParams(ctypes.Structure):
    _fields_ = [
        ("tau", c_double),
        ("sigma_a", c_double),
        ("sigma_s", c_double),
        ("phase_g", c_double),
        ("gather_dist", c_double),
        ("scattering", c_int32),
        ("n_scat", c_int32),
    ]


class FvrLoopState(ctypes.Structure):
    _fields_ = [
        ("it", c_int32),
        ("done", c_int32),
        ("converged", c_int32),
        ("reserved", c_int32),
        ("prev_rmse", c_double),
        ("work_next", c_int32),
        ("work_retired", c_int32),
    ]


class FvrLoopFinalize(ctypes.Structure):
    _fields_ = [
        ("n_views", c_int32),
        ("blocks_per_view", c_int32),
        ("pixels_per_view", c_int64),
        ("vol_partials", c_void_p),
        ("n_vol_blocks", c_int32),
        ("reserved", c_int32),
        ("n_kp", c_int64),
        ("converge_eps", c_double),
        ("trace_rmse", c_void_p),
        ("trace_vol", c_void_p),
        ("trace_stride", c_int64),
        ("sq_accum", c_void_p),
        ("l2_discard", c_void_p),
        ("l2_discard_bytes", c_int64),
    ]


_P = c_void_p  # every pointer argument is passed as an address
_GRID = FvrGrid
_PARAMS = FvrRenderParams

# name -> (restype, argtypes); mirrors include/fvr_b200.h
_SIGNATURES = {
    "fvr_last_error": (c_char_p, []),
    "fvr_abi_version": (c_int, []),
    "fvr_launch_count": (c_int64, []),
    "fvr_render_rays": (c_int, [_P, _P, c_int64, _P, c_int32, _GRID, _PARAMS, _P, _P, _P, _P, _P, _P]),
    "fvr_render_rays_host": (c_int, [_P, _P, c_int64, _P, c_int32, _GRID, _PARAMS, _P, _P, _P]),
    "fvr_count_hull_samples": (c_int, [_P, _P, c_int64, _P, _GRID, _P, _P]),
    "fvr_count_hull_samples_host": (c_int, [_P, _P, c_int64, _P, _GRID, _P]),
    "fvr_adjust_rays": (
        c_int,
        [_P, _P, c_int64, _P, _P, _P, c_int32, _P, _GRID, c_double, c_double, c_double, _P, _P],
    ),
    "fvr_adjust_rays_host": (
        c_int,
        [_P, _P, c_int64, _P, _P, _P, c_int32, _P, _GRID, c_double, c_double, c_double, _P, c_int32],
    ),
    "fvr_apply_correction": (c_int, [_P, _P, _P, c_int64, _P]),
    "fvr_render_pixels": (
        c_int,
        [_P, _P, _P, c_int64, _P, c_int32, _GRID, _PARAMS, _P, _P, _P, _P, _P, _P],
    ),
    "fvr_occupancy": (c_int, [_P, c_int32, _P, _GRID, _P, _P]),
    "fvr_render_views": (
        c_int, [_P, c_int32, c_int32, c_int32, _P, c_int32, _GRID, _PARAMS, _P, _P, _P, _P, _P, _P]),
    "fvr_set_scatter_dirs": (c_int, [_P, c_int32]),
    "fvr_render_layout_kind": (c_int, [_PARAMS, _GRID]),
    "fvr_pack_layout": (c_int, [_P, c_int32, _GRID, c_int32, _P, _P]),
    "fvr_loop_blocks_per_view": (c_int, [c_int32, c_int32]),
    "fvr_loop_render": (
        c_int,
        [_P, c_int32, c_int32, c_int32, c_int32, c_int32, _P, _P, _P, _P, _GRID, _PARAMS, _P, c_int32, _P,
         _P, _P, c_int64, _P, _P],
    ),
    "fvr_loop_adjust": (
        c_int,
        [_P, _P, c_int64, c_int32, c_int32, c_int32, c_int32, _P, c_int32, _P, _GRID, c_double, c_double,
         c_double, c_int32, c_double, c_uint64, c_int64, _P, _P, _P],
    ),
    "fvr_loop_volume_sq": (c_int, [_P, _P, _P, c_int64, _P, POINTER(c_int32), _P, _P]),
    "fvr_loop_finalize": (
        c_int,
        [_P, c_int32, c_int32, c_int64, _P, c_int32, c_int64, c_double, _P, _P, _P, _P],
    ),
    "fvr_loop_update": (c_int, [_P, _P, _P, c_int64, _P, c_int32, c_int32, _GRID, _P, _P]),
    "fvr_adjust_plan_count": (
        c_int, [_P, _P, c_int64, c_int32, c_int32, c_int32, c_int32, _P, _GRID, _P, _P, _P]),
    "fvr_adjust_plan_fill": (
        c_int, [_P, _P, c_int64, c_int32, c_int32, c_int32, c_int32, _P, _GRID, c_double, c_double, c_double,
                _P, _P, _P, _P, _P, _P]),
    "fvr_rplan_chunk_entries": (c_int, []),
    "fvr_rplan_count": (c_int, [_P, c_int32, c_int32, c_int32, c_int32, c_int32, _GRID, _PARAMS, _P, _P, _P, _P,
                                _P]),
    "fvr_rplan_fill": (c_int, [_P, c_int32, c_int32, c_int32, c_int32, c_int32, _GRID, _PARAMS, _P, _P, _P, c_int32,
                               _P, _P, _P, _P, _P, _P, _P, _P, _P, c_int32, _P]),
    "fvr_rplan_pos27": (c_int, [_GRID, _P, _P, c_int32, _P, _P]),
    "fvr_rplan_unit_keys": (c_int, [_P, c_int32, c_int32, c_int32, c_int32, _P, _P, _P]),
    "fvr_rplan_render": (c_int, [_P, _P, _P, _P, _P, _P, _P, _P, c_int32, c_int32, c_int32, _P, _P, c_int32, _P, _P,
                                 _P, c_int64, _P, _P, c_int32, _P]),
    "fvr_rplan_pack": (c_int, [_P, c_int32, _GRID, _P, c_int64, _P, _P, _P]),
    "fvr_sample_plan_count": (c_int, [_P, _P, c_int64, c_int32, c_int32, c_int32, c_int32, _P, _GRID, _P, _P, _P,
                                      _P]),
    "fvr_sample_plan_fill": (c_int, [_P, _P, c_int64, c_int32, c_int32, c_int32, c_int32, _P, _GRID, c_double,
                                     c_double, c_double, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "fvr_sample_plan_reorder": (c_int, [_P, c_int64, c_int32, _P, c_int64, _P, _P, _P]),
    "fvr_loop_weighted_residual": (c_int, [_P, c_int64, _P, c_int32, c_int32, _P, c_int32, c_uint64, c_double,
                                           c_int64, _P, _P, c_int32, _P]),
    "fvr_stochastic_g": (c_int, [c_uint64, ctypes.c_uint32, _P, _P, c_int64, c_double, _P, _P]),
    "fvr_loop_gather": (c_int, [_P, _P, _P, _P, _P, c_int64, _P, c_int32, _P, _P, _P, c_int32, _GRID, _P, _P, _P,
                                c_int32, _P]),
    "fvr_loop_update_packed": (c_int, [_P, c_int64, _P, _P, _P, c_int32, c_int32, _GRID, _P, c_int32, _P, _P]),
    "fvr_pack_correction": (c_int, [_P, _P, c_int64, _P, _P]),
    "fvr_unpack_correction": (c_int, [_P, _P, c_int64, _P, _P]),
    "fvr_ctmap_build": (c_int, [c_double, c_double, c_int32, c_int32, c_double, _P, _P, _P]),
    "fvr_temp_lookup": (c_int, [_P, _P, c_int64, _P, _P, c_int32, _P, _P, _P, _P]),
    "fvr_temp_from_green": (c_int, [_P, c_int64, _P, _P, c_int32, _P, _P, _P]),
    "fvr_temp_rgb": (c_int, [_P, _P, c_int64, _P, _P, _P, c_int32, _P, _P, c_int64, _P, _P]),
    "fvr_visual_hull_view": (c_int, [_P, _P, _GRID, _P, c_int32, _P, _P]),
    "fvr_hull_keypoints": (c_int, [_P, _GRID, _P, _P, _P]),
    "fvr_threshold_mask": (c_int, [_P, c_int32, c_int32, c_int32, c_int32, c_double, _P, _P, _P, _P]),
    "fvr_mask_sat": (c_int, [_P, c_int32, c_int32, _P, _P]),
    "fvr_stage_inputs_host": (c_int, [_P, c_int64, ctypes.c_uint32, c_int32, _P, _P, c_int64, _P, _P, c_int32, c_int32,
                                      c_int32, c_int32, _P, _P, _P, _P]),
    "fvr_morton_keys": (c_int, [_P, c_int64, _GRID, _P, _P]),
    "fvr_sell_window_order": (c_int, [_P, c_int64, c_int32, _P, _P]),
    "fvr_rplan_tile_rows": (c_int, [_P, c_int32, c_int32, c_int32, c_int32, c_int32, c_int32, _P, _P, _P]),
    "fvr_morton_order": (c_int, [_P, c_int64, _GRID, _P, _P]),
    "fvr_kp_map": (c_int, [_P, c_int64, c_int64, _P, _P]),
    "fvr_sell_layout": (c_int, [_P, c_int64, c_int32, c_int32, _P, c_int64, _P, _P, _P, _P, _P, _P, _P]),
    "fvr_sample_plan_spatial": (c_int, [_P, c_int64, c_int32, _P, c_int64, _P, _P, _P]),
    "fvr_plan_sort_rows": (c_int, [_P, _P, c_int64, _P, _P, _P]),
    "fvr_sell_pad_zero": (c_int, [_P, _P, c_int64, _P, _P, c_int64, _P, _P, _P]),
    "fvr_count_nonzero_u8": (c_int, [_P, c_int64, _P, _P]),
    "fvr_copy_host_parallel": (c_int, [_P, _P, c_int32, _P]),
    "fvr_select_nonzero_u8": (c_int, [_P, c_int64, c_int64, _P, _P, _P]),
    "fvr_rplan_layout": (c_int, [_P, c_int32, c_int32, c_int32, c_int32, c_int32, c_int32, c_int32, _P, _P, _P, _P,
                                 _P, _P]),
    "fvr_flame_rays": (c_int, [_P, c_int32, c_int32, c_int32, c_int64, _P, _P, _P]),
    "fvr_comm_available": (c_int, []),
    "fvr_comm_nccl_version": (c_int, [POINTER(c_int32)]),
    "fvr_comm_unique_id": (c_int, [_P]),
    "fvr_comm_init": (c_int, [c_int32, c_int32, _P, c_int32, POINTER(c_void_p)]),
    "fvr_allreduce_sum": (c_int, [c_void_p, _P, c_int64, c_int32, _P]),
    "fvr_comm_destroy": (c_int, [c_void_p]),
}

FVR_COMM_ID_BYTES = 128
FVR_DT_INT64, FVR_DT_FLOAT32, FVR_DT_FLOAT64 = 0, 1, 2

EXPORTED_SYMBOLS = tuple(_SIGNATURES)

_lib = None


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load the shared library (no CUDA calls happen at load time)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(
            f"libfvr_b200.so not found at {path}; build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)"
        )
    lib = ctypes.CDLL(path)
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int) -> None:
    """Map a C-ABI status to the reference's exception types."""
    if rc == FVR_OK:
        return
    msg = load().fvr_last_error().decode("utf-8", "replace")
    if rc == FVR_ERR_INVALID:
        raise ValueError(msg)
    if rc == FVR_ERR_EMPTY_HULL:
        raise EmptyHullError(msg)
    if rc == FVR_ERR_NO_FLAME:
        raise NoFlameError(msg)
    raise RuntimeError(f"libfvr_b200: {msg}")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))


def launch_count() -> int:
    return int(load().fvr_launch_count())


# --- torch handoff ------------------------------------------------------------

_torch = None


def torch():
    """Import torch lazily (it is plumbing: device memory and streams)."""
    global _torch
    if _torch is None:
        import torch as _t

        _torch = _t
    return _torch


def device():
    t = torch()
    if not t.cuda.is_available():
        raise RuntimeError(
            "paper_1809_06417_b200 needs a CUDA device (sm_100a); there is no CPU fallback"
        )
    load()
    return t.device("cuda", t.cuda.current_device())


class nvtx:
    """NVTX range around a host-side stage (the C-ABI entry points carry their
    own ranges); a no-op cost when no profiler is attached."""

    def __init__(self, name: str):
        self.name = name

    def __enter__(self):
        torch().cuda.nvtx.range_push(self.name)
        return self

    def __exit__(self, *exc):
        torch().cuda.nvtx.range_pop()
        return False


def stream_ptr() -> int:
    return torch().cuda.current_stream().cuda_stream


def ptr(tensor) -> int | None:
    if tensor is None:
        return None
    return tensor.data_ptr()


def grid_struct(grid) -> FvrGrid:
    g = FvrGrid()
    g.nx, g.ny, g.nz = int(grid.nx), int(grid.ny), int(grid.nz)
    g.reserved = 0
    for a in range(3):
        g.origin[a] = float(grid.origin[a])
    g.edge = float(grid.edge)
    return g


def camera_struct(cam) -> FvrCamera:
    c = FvrCamera()
    c.fx, c.fy, c.cx, c.cy = float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy)
    R = cam.rotation.ravel()
    for i in range(9):
        c.rotation[i] = float(R[i])
    ctr = cam.center  # -R^T t, computed by numpy exactly as the reference
    for a in range(3):
        c.center[a] = float(ctr[a])
    c.width, c.height = int(cam.width), int(cam.height)
    return c


def to_host(tensor):
    """D2H of a device tensor through page-locked memory (torch's caching host
    allocator): several times a pageable .cpu() for the tens-of-MB lattices
    of the larger configs.  Returns a numpy array viewing the pinned buffer."""
    t = torch()
    host = t.empty(tuple(tensor.shape), dtype=tensor.dtype, pin_memory=True)
    host.copy_(tensor, non_blocking=True)
    t.cuda.current_stream().synchronize()
    return host.numpy()


class HostRead:
    """A small D2H queued now on the current stream into page-locked memory,
    read later: ``get()`` waits for this copy only (an event), so the host can
    queue other work while the device catches up."""

    def __init__(self, tensor):
        t = torch()
        self.host = t.empty(tuple(tensor.shape), dtype=tensor.dtype, pin_memory=True)
        self.host.copy_(tensor, non_blocking=True)
        self.event = t.cuda.Event()
        self.event.record()

    def get(self):
        self.event.synchronize()
        return self.host.tolist()


def upload_host(arrays, dtype, shape, dev):
    """Host arrays concatenated (fvr_copy_host_parallel, all host threads) into
    page-locked staging, then one asynchronous H2D into a new device tensor of
    ``shape``."""
    import numpy as np

    t = torch()
    arrs = [np.ascontiguousarray(a) for a in arrays]
    nbytes = [a.nbytes for a in arrs]
    total = sum(nbytes)
    stage = t.empty(total, dtype=t.uint8, pin_memory=True)
    n = len(arrs)
    srcs = (ctypes.c_void_p * n)(*[a.ctypes.data for a in arrs])
    sizes = (ctypes.c_int64 * n)(*nbytes)
    call("fvr_copy_host_parallel", ctypes.addressof(srcs), ctypes.addressof(sizes), n, stage.data_ptr())
    out = t.empty(total, dtype=t.uint8, device=dev)
    out.copy_(stage, non_blocking=True)  # (the caching host allocator keeps stage until the copy is done)
    return out.view(dtype).view(shape)


def cameras_tensor(cameras, dev):
    """Pack cameras into a device byte tensor holding fvr_camera_t[V]."""
    t = torch()
    n = len(cameras)
    arr = (FvrCamera * n)(*[camera_struct(c) for c in cameras])
    host = t.frombuffer(bytearray(bytes(arr)), dtype=t.uint8)
    return host.to(dev)


_dirs_loaded = False


def ensure_scatter_dirs() -> None:
    """Load fibonacci_sphere(32) into the stencil path's constant memory (once)."""
    global _dirs_loaded
    if _dirs_loaded:
        return
    import numpy as np

    from .radiometry import fibonacci_sphere

    d = np.ascontiguousarray(fibonacci_sphere(32))
    call("fvr_set_scatter_dirs", d.ctypes.data, 32)
    _dirs_loaded = True


def layout_kind(params: FvrRenderParams, grid: FvrGrid) -> int:
    """0 (none), 1 (YZQ) or 2 (Z4): the packed layout the fast render path reads."""
    ensure_scatter_dirs()
    return int(load().fvr_render_layout_kind(params, grid))


def render_params(cfg, scattering: bool, n_scat: int, phase_g: float, gather: float) -> FvrRenderParams:
    p = FvrRenderParams()
    p.tau = float(cfg.tau)
    p.sigma_a = float(cfg.sigma_a)
    p.sigma_s = float(cfg.sigma_s)
    p.phase_g = float(phase_g)
    p.gather_dist = float(gather)
    p.scattering = 1 if scattering else 0
    p.n_scat = int(n_scat)
    return p
