#!/bin/bash
# A/B of library builds on one BASELINE config's device loop (ms per iteration):
#   tools/ab_config.sh 4 libfvr_b200.so libfvr_b200_x.so ...
cfg=$1; shift
python - "$cfg" "$@" <<'PY'
import os, sys, subprocess, json
cfg = sys.argv[1]
for lib in sys.argv[2:]:
    code = f"""
import os, sys, json
sys.path.insert(0, '.')
import torch
torch.cuda.set_device(0)
import workloads
from tools.config_baselines import gpu_loop
sc = workloads.device_scene(*workloads.CONFIGS[{cfg}])
for _ in range(2):
    r = gpu_loop(sc)
    print(json.dumps({{'lib': '{lib}', 'ms_per_iter': r['ms_per_iter'], 'setup_s': r['setup_s']}}))
"""
    out = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, FVR_LIB=lib), capture_output=True, text=True)
    print(out.stdout.strip() or out.stderr[-800:], flush=True)
PY
