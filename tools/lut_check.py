import sys; sys.path.insert(0, ".")
import numpy as np, time, torch
from tests.conftest import load_golden
from paper_1809_06417_b200 import build_color_temp_map
g = load_golden("ctmap.npz")
cmap = build_color_temp_map(1000.0, 2300.0, 1.0)
print("exact frac", np.mean(cmap.entries == g["entries"]), "n diff", int((cmap.entries != g["entries"]).sum()), cmap.entries.size)
d = np.abs(cmap.entries - g["entries"]) / np.maximum(np.abs(g["entries"]), 1e-300)
print("max rel", d.max())
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5): build_color_temp_map(1000.0, 2300.0, 1.0)
torch.cuda.synchronize()
print("build ms", (time.perf_counter() - t0) / 5 * 1e3)
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    build_color_temp_map(1000.0, 2300.0, 1.0)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=12))
print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=12))
