#!/bin/bash
# Round-2 artefact refresh on one GPU: bench line, reference arm, launch lists
# (the timed region via its NVTX range, and the whole bench), full ncu
# captures of the loop kernels and of the setup kernels.  Outputs land in
# gpurun_out/r2final/ (summaries copied to profiles/ by hand).
set -u
O=gpurun_out/r2final
mkdir -p $O
python bench.py > $O/bench.json 2> $O/bench.err
python bench.py --impl reference > $O/ref.json 2> $O/ref.err
ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/launches_timed.csv \
    python bench.py --steps 5 --warmup 3 --e2e-iters 0 --no-cpu-baseline --stochastic-steps 5 > $O/ncu_timed.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_all.csv \
    python bench.py --steps 5 --warmup 3 --e2e-iters 0 --no-cpu-baseline --stochastic-steps 5 > $O/ncu_all.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"rplan_render|gather_kernel" -s 4 -c 2 \
    -o $O/prof_det python bench.py --steps 3 --warmup 3 --e2e-iters 0 --no-cpu-baseline --stochastic-steps 0 \
    > $O/ncu_det.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"weighted_residual|gather_kernel" -s 6 -c 2 \
    -o $O/prof_sto python bench.py --steps 3 --warmup 3 --e2e-iters 0 --no-cpu-baseline --stochastic-steps 3 \
    > $O/ncu_sto.log 2>&1
ncu --set full --import-source on --clock-control none \
    -k regex:"rplan_fill_kernel|plan_fill_kernel|rplan_count_kernel|plan_count_kernel" -c 4 \
    -o $O/prof_fill python tools/profile_setup.py > $O/ncu_fill.log 2>&1
ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k regex:"weighted_residual|gather_kernel<0, 1, 1, 0>" -c 2 \
    -o $O/prof_sto2 python bench.py --steps 3 --warmup 3 --e2e-iters 0 --no-cpu-baseline --stochastic-steps 3 \
    > $O/ncu_sto2.log 2>&1
ls -la $O
