"""Where ChannelLoop setup time goes at config 2: every C-ABI call timed with
a device synchronize on both sides (so the sum is serialised device + host
time), plus the wall time of the whole reconstruct_channel call."""
import collections
import sys
import time

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1809_06417_b200 import ReconstructionConfig, _lib, reconstruct_channel  # noqa: E402
from paper_1809_06417_b200 import engine  # noqa: E402

sc = bench.make_scene()
cfg = ReconstructionConfig(alpha_l=bench.ALPHA_L, alpha_d=1.0, tau=bench.TAU, max_iters=50,
                           converge_eps=1e-12, deterministic_mode=True)
t = _lib.torch()


def call():
    return reconstruct_channel(sc["images"], sc["cams"], sc["geom"], sc["hull"], cfg, render_cfg=sc["rcfg"],
                               masks=sc["masks"], bbox=sc["bbox"])


for _ in range(3):
    call()
for _ in range(3):
    t0 = time.perf_counter()
    call()
    print(f"wall {1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)

acc = collections.defaultdict(float)
orig_call = _lib.call


def timed(name, *args):
    t.cuda.synchronize()
    t0 = time.perf_counter()
    orig_call(name, *args)
    t.cuda.synchronize()
    acc[name] += (time.perf_counter() - t0) * 1e3


orig_init = engine.ChannelLoop.__init__


def init(self, *a, **k):
    t.cuda.synchronize()
    t0 = time.perf_counter()
    orig_init(self, *a, **k)
    t.cuda.synchronize()
    acc["__init__ total"] += (time.perf_counter() - t0) * 1e3


_lib.call = timed
engine._lib.call = timed
engine.ChannelLoop.__init__ = init
t0 = time.perf_counter()
call()
acc["reconstruct_channel total (synced calls)"] = (time.perf_counter() - t0) * 1e3
for k, v in sorted(acc.items(), key=lambda kv: -kv[1]):
    print(f"{v:8.3f} ms  {k}")

# section marks inside ChannelLoop.__init__ (host ms = when the host got there)
import os  # noqa: E402

_lib.call = orig_call
engine._lib.call = orig_call
engine.ChannelLoop.__init__ = orig_init
os.environ["FVR_INIT_PROFILE"] = "1"
captured = []
orig_run = engine.ChannelLoop.run


def run(self, *a, **k):
    captured.append(self)
    return orig_run(self, *a, **k)


engine.ChannelLoop.run = run
t_init = []


def init2(self, *a, **k):
    t_init.append(time.perf_counter())
    orig_init(self, *a, **k)
    t_init.append(time.perf_counter())


engine.ChannelLoop.__init__ = init2
for _ in range(2):
    captured.clear()
    t_init.clear()
    t0 = time.perf_counter()
    call()
    t1 = time.perf_counter()
    print(f"call wall {1e3 * (t1 - t0):.2f} ms: before ChannelLoop {1e3 * (t_init[0] - t0):.2f} ms, "
          f"__init__ {1e3 * (t_init[1] - t_init[0]):.2f} ms, after {1e3 * (t1 - t_init[1]):.2f} ms")
    for name, host_ms, dev_ms in captured[0].init_profile():
        print(f"  {name:18s} host {host_ms:7.3f} ms   device {dev_ms:7.3f} ms")
