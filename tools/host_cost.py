"""Host-side cost (no synchronisation) of the setup's native layout calls at
config 2 sizes: each call timed with perf_counter around the ctypes call."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1809_06417_b200 import _lib  # noqa: E402

torch.cuda.set_device(0)
dev = torch.device("cuda:0")
n_views, w, h = 8, 139, 255
ux, uy = (w + 7) // 8, (h + 3) // 4
n_units = n_views * ux * uy
row_len = torch.randint(0, 600, (n_units * 32,), dtype=torch.int32, device=dev)
counts = torch.randint(0, 200, (306607,), dtype=torch.int32, device=dev)
kp = torch.randint(0, 129 ** 3, (306607,), dtype=torch.int32, device=dev)
mask = (torch.rand(129 ** 3, device=dev) < 0.15).to(torch.uint8)
g = _lib.FvrGrid()
g.nx = g.ny = g.nz = 128
g.edge = 1.0
st = _lib.stream_ptr()


def timed(name, fn, reps=20):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
        torch.cuda.synchronize()
    print(f"{name:28s} host {1e6 * np.median(ts):8.1f} us")


def rplan_layout():
    row_src = torch.empty(n_units * 32, dtype=torch.int32, device=dev)
    unit_len = torch.empty(n_units, dtype=torch.int32, device=dev)
    off = torch.empty(n_units + 1, dtype=torch.int64, device=dev)
    order = torch.empty(n_units, dtype=torch.int32, device=dev)
    totals = torch.empty(2, dtype=torch.int64, device=dev)
    _lib.call("fvr_rplan_layout", row_len.data_ptr(), n_views, w, h, 2, 4, 16, 24, row_src.data_ptr(),
              unit_len.data_ptr(), off.data_ptr(), order.data_ptr(), totals.data_ptr(), st)


def sell_layout():
    n = counts.numel()
    ns = (n + 31) // 32
    a = torch.empty(n, dtype=torch.int32, device=dev)
    b = torch.empty(ns, dtype=torch.int32, device=dev)
    c = torch.empty(ns + 1, dtype=torch.int64, device=dev)
    d = torch.empty(n, dtype=torch.int64, device=dev)
    tot = torch.empty(3, dtype=torch.int64, device=dev)
    _lib.call("fvr_sell_layout", counts.data_ptr(), n, 128, 8, None, 0, None, a.data_ptr(), b.data_ptr(),
              c.data_ptr(), d.data_ptr(), tot.data_ptr(), st)


def morton():
    out = torch.empty_like(kp)
    _lib.call("fvr_morton_order", kp.data_ptr(), kp.numel(), g, out.data_ptr(), st)


def select():
    cnt = torch.empty(1, dtype=torch.int64, device=dev)
    out = torch.empty(400000, dtype=torch.int32, device=dev)
    _lib.call("fvr_select_nonzero_u8", mask.data_ptr(), mask.numel(), 400000, out.data_ptr(), cnt.data_ptr(), st)


def empty5():
    for _ in range(5):
        torch.empty(100000, dtype=torch.int32, device=dev)


def event():
    e = torch.cuda.Event()
    e.record()


timed("fvr_rplan_layout", rplan_layout)
timed("fvr_sell_layout", sell_layout)
timed("fvr_morton_order", morton)
timed("fvr_select_nonzero_u8", select)
timed("5 x torch.empty", empty5)
timed("event record", event)
