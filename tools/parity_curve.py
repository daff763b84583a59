"""Max-error-per-iteration curve of the device loop against the CPU oracle on
identical full-size inputs (profiles/r2_parity_curve_*.json).

  python tools/parity_curve.py CONFIG ITERS [modes=plan,march] [out.json]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from tests.fullsize_common import curve, device_loop, oracle_loop  # noqa: E402
from workloads import CONFIGS, device_scene  # noqa: E402


def main():
    cfg_no, iters = int(sys.argv[1]), int(sys.argv[2])
    modes = (sys.argv[3] if len(sys.argv) > 3 else "plan,march").split(",")
    out = sys.argv[4] if len(sys.argv) > 4 else f"gpurun_out/parity_curve_c{cfg_no}.json"
    torch.cuda.set_device(0)
    n, views, res = CONFIGS[cfg_no]
    t0 = time.perf_counter()
    sc = device_scene(n, views, res)
    res_ = {"config": cfg_no, "n": n, "views": views, "res": res, "iters": iters, "scene_s": time.perf_counter() - t0}
    devs = {}
    for m in modes:
        t0 = time.perf_counter()
        devs[m] = device_loop(sc, iters, m)
        res_[f"device_{m}_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    ref = oracle_loop(sc, iters)
    res_["oracle_s"] = time.perf_counter() - t0
    res_["oracle_s_per_iter"] = ref[3]
    res_["cores"] = os.cpu_count()
    for m in modes:
        res_[m] = curve(devs[m], ref)
        print(m, "final", res_[m]["final_grid_rel"], "max per-iter", max(res_[m]["grid_rel_per_iter"]),
              "rmse rel max", max(res_[m]["rmse_rel_per_iter"]), flush=True)
    os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
    with open(out, "w") as f:
        json.dump(res_, f)
    print(json.dumps({k: v for k, v in res_.items() if not isinstance(v, dict)}))


if __name__ == "__main__":
    main()
