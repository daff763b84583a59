"""Device timeline of one public-API reconstruct_channel call (config 2, 50
iterations) from the CUDA activity trace (torch.profiler / CUPTI): every
kernel and copy with its start, duration and stream, relative to the call's
first device activity.  python tools/e2e_trace.py [out.txt]"""
import json
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
from paper_1809_06417_b200 import ReconstructionConfig, reconstruct_channel  # noqa: E402

torch.cuda.set_device(0)
sc = bench.make_scene()
cfg = ReconstructionConfig(alpha_l=bench.ALPHA_L, alpha_d=1.0, tau=bench.TAU, max_iters=50, converge_eps=1e-12,
                           deterministic_mode=os.environ.get("E2E_STOCHASTIC") != "1", g_sigma=0.1, rng_seed=0)


def call():
    reconstruct_channel(sc["images"], sc["cams"], sc["geom"], sc["hull"], cfg, render_cfg=sc["rcfg"],
                        masks=sc["masks"], bbox=sc["bbox"])


for _ in range(4):
    call()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    call()
    torch.cuda.synchronize()
path = os.path.join(tempfile.mkdtemp(), "trace.json")
prof.export_chrome_trace(path)
ev = json.load(open(path))["traceEvents"]
dev = [e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
cpu = [e for e in ev if e.get("ph") == "X" and e.get("cat") == "cpu_op"]
t0 = min(e["ts"] for e in dev)
t_end = max(e["ts"] + e["dur"] for e in dev)
out = [f"device span {1e-3 * (t_end - t0):.3f} ms, {len(dev)} device activities"]
busy = 0.0
last = t0
for e in sorted(dev, key=lambda e: e["ts"]):
    s, d = e["ts"] - t0, e["dur"]
    busy += max(0.0, min(e["ts"] + d, t_end) - max(e["ts"], last))
    last = max(last, e["ts"] + d)
    if e["cat"] != "kernel" or not any(k in e["name"] for k in ("rplan_render", "gather_kernel")):
        out.append(f"{s / 1e3:8.3f} ms  {d / 1e3:7.3f} ms  s{e['args'].get('stream', '?')}  {e['name'][:90]}")
out.append(f"device busy {busy / 1e3:.3f} ms of {1e-3 * (t_end - t0):.3f} ms")
loop = [e for e in dev if any(k in e["name"] for k in ("rplan_render", "gather_kernel"))]
if loop:
    ls = min(e["ts"] for e in loop) - t0
    le = max(e["ts"] + e["dur"] for e in loop) - t0
    out.append(f"loop kernels {len(loop)}: from {ls / 1e3:.3f} to {le / 1e3:.3f} ms ({(le - ls) / 1e3:.3f} ms)")
text = "\n".join(out)
print(text)
if len(sys.argv) > 1:
    open(sys.argv[1], "w").write(text + "\n")
