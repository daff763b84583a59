#!/bin/bash
# Stochastic sample-plan rows sorted by sample id (FVR_SPLAN_SORT) vs not:
# loop stage times, the stochastic public-API call, and the stochastic tests
mkdir -p gpurun_out
bash tools/ab_env.sh "FVR_SPLAN_SORT=1" "FVR_SPLAN_SORT=0" > gpurun_out/ab_rowsort_bench.txt 2>&1
for cfg in FVR_SPLAN_SORT=1 FVR_SPLAN_SORT=0; do
  env $cfg python bench.py --no-cpu-baseline --e2e-iters 0 --steps 50 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); s=d['stochastic']; print('$cfg', round(s['value'],1), s['stage_ms'])" >> gpurun_out/ab_rowsort_bench.txt
done
E2E_STOCHASTIC=1 python tools/e2e_ab.py 12 base,no_row_sort > gpurun_out/ab_rowsort_e2e.txt 2>&1
python -m pytest tests/test_gpu_stochastic.py tests/test_gpu_loop_features.py -q -x -m gpu > gpurun_out/ab_rowsort_pytest.log 2>&1
tail -1 gpurun_out/ab_rowsort_pytest.log
