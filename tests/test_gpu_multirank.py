"""The device ChannelLoop at world size 2 and 3 on one B200 (§8e view
sharding): each rank renders and back-projects its own views, and the
exchange all-reduces the i64 [packed correction | RMSE partials] buffer.

The ranks are processes on cuda:0 with the gloo transport, whose all-reduce
stages CUDA tensors through the host: no kernel ever waits on another rank
(the NCCL path needs one GPU per rank; it runs at world size 1 in
test_nccl_comm_single_rank).  Grids and traces must be bit-identical to the
unsharded loop in deterministic and stochastic mode: corrections are 32.32
fixed-point integers and each f64 partial has exactly one owner.  The
reference behaviour being sharded is the per-view loop and fixed-order merge
of adjust_pass (reconstruct.py:181-226)."""

import multiprocessing as mp
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _loop(fixture: str, deterministic: bool, iters: int, rgb: bool = False):
    from paper_1809_06417_b200 import ReconstructionConfig, reconstruct_channel, reconstruct_color
    from tests.conftest import load_golden
    from tests.test_gpu_parity import _loop_inputs

    g = load_golden(fixture)
    cams, hull, images, masks, bbox, geom, rcfg = _loop_inputs(g)
    cfg = ReconstructionConfig(alpha_l=0.006, alpha_d=1.0, tau=float(g["tau"]), max_iters=iters,
                               converge_eps=1e-12, deterministic_mode=deterministic, g_sigma=0.1, rng_seed=3)
    if rgb:
        from paper_1809_06417_b200.imgio import Image

        rgb_imgs = [Image(im.shape[1], im.shape[0], 3, im) for im in g["images"]]
        res = reconstruct_color(rgb_imgs, cams, geom, cfg, render_cfg=rcfg)
        return np.stack([gr.values for gr in res.grids]), [res.traces[t].rmse for t in ("red", "green", "blue")]
    grid, trace = reconstruct_channel(images, cams, geom, hull, cfg, render_cfg=rcfg, masks=masks, bbox=bbox)
    return grid.values, trace.rmse


def _rank(rank: int, world: int, port: int, case, q) -> None:
    try:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(0)
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        try:
            vals, rmse = _loop(*case)
            q.put((rank, vals, rmse, None))
        finally:
            dist.destroy_process_group()
    except Exception as e:  # report instead of hanging the parent
        import traceback

        q.put((rank, None, None, traceback.format_exc() + repr(e)))


def _sharded(case, world: int):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        r, vals, rmse, err = q.get(timeout=600)
        assert err is None, err
        out[r] = (vals, rmse)
    for p in procs:
        p.join(timeout=60)
    return out


CASES = [("config1.npz", True, 10), ("config1.npz", False, 10), ("loop_scatter.npz", True, 5),
         ("loop_scatter.npz", False, 5)]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0][:-4]}-{'det' if c[1] else 'stoch'}")
@pytest.mark.parametrize("world", [2, 3])
def test_sharded_loop_is_bit_identical(cuda_device, case, world):
    one_vals, one_rmse = _loop(*case)
    out = _sharded(case, world)
    for r in range(world):
        vals, rmse = out[r]
        assert np.array_equal(vals, one_vals), (r, float(np.max(np.abs(vals - one_vals))))
        assert list(rmse) == list(one_rmse)


def test_sharded_rgb_loop_is_bit_identical(cuda_device):
    case = ("config1.npz", True, 6, True)
    one_vals, one_rmse = _loop(*case)
    out = _sharded(case, 2)
    for r in range(2):
        vals, rmse = out[r]
        assert np.array_equal(vals, one_vals)
        assert [list(x) for x in rmse] == [list(x) for x in one_rmse]


def _nccl_rank(port: int, q) -> None:
    try:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(0)
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
        os.environ["FVR_FORCE_SHARDED"] = "1"
        from paper_1809_06417_b200 import _lib
        from paper_1809_06417_b200.engine import DeviceComm, _collective

        dc = _collective()
        assert isinstance(dc, DeviceComm)
        import ctypes

        ver = ctypes.c_int32(0)
        _lib.call("fvr_comm_nccl_version", ctypes.byref(ver))
        v = int(ver.value)
        buf = torch.arange(1000, dtype=torch.int64, device="cuda") - 500
        want = buf.clone()
        dc.allreduce_sum_(buf, _lib.stream_ptr())
        torch.cuda.synchronize()
        ok = bool(torch.equal(buf, want))
        vals, rmse = _loop("config1.npz", True, 10)
        dist.destroy_process_group()
        q.put((v, ok, vals, rmse, None))
    except Exception as e:
        import traceback

        q.put((None, False, None, None, traceback.format_exc() + repr(e)))


def test_nccl_comm_single_rank(cuda_device):
    """fvr_comm_init / fvr_allreduce_sum on a 1-rank NCCL group, and the
    loop's sharded stages driven through it (FVR_FORCE_SHARDED)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_rank, args=(_free_port(), q))
    p.start()
    v, ok, vals, rmse, err = q.get(timeout=600)
    p.join(timeout=60)
    assert err is None, err
    assert v is not None and v >= 22000, v
    assert ok
    one_vals, one_rmse = _loop("config1.npz", True, 10)
    assert np.array_equal(vals, one_vals)
    assert list(rmse) == list(one_rmse)


def test_bench_two_ranks_plumbing(cuda_device):
    """bench.py --gpus 2 relaunches itself under torchrun, shards the views,
    times max-over-ranks and prints ONE line from rank 0 (ranks on cuda:0 over
    gloo here: FVR_BENCH_ONE_GPU; the driver's multi-GPU run uses NCCL)."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, FVR_BENCH_ONE_GPU="1")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--steps", "3", "--warmup",
                          "3", "--e2e-iters", "4", "--stochastic-steps", "2", "--no-cpu-baseline"],
                         cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == 2 and rec["value"] > 0 and rec["config"]["parallelism"] == "view-sharded x2"
    assert rec["e2e"]["value"] > 0 and rec["stochastic"]["value"] > 0
