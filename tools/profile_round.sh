#!/bin/bash
# One GPU session that refreshes every judged artefact: bench line, the other
# configs, the render sweep, the launch list and full ncu captures of the
# loop kernels.  Outputs land in gpurun_out/final/ (copied to profiles/ by hand).
set -u
O=gpurun_out/final
mkdir -p $O
python bench.py > $O/bench.json 2> $O/bench.err
python tools/rgb_bench.py > $O/rgb.json 2> $O/rgb.err
python tools/run_configs.py 3 20 > $O/config3.json 2> $O/config3.err
python tools/run_configs.py 4 10 > $O/config4.json 2> $O/config4.err
timeout 900 python tools/run_configs.py sweep > $O/sweep.jsonl 2> $O/sweep.err
# launch list of the bench command (cold-cache, serialised: shares, not absolutes)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py --steps 5 --warmup 3 --e2e-iters 0 --no-cpu-baseline --stochastic-steps 5 > $O/ncu_launch.log 2>&1
# full captures: deterministic render + gather, then the stochastic weigh + sample-plan gather
ncu --set full --import-source on --clock-control none -k regex:"rplan_render|gather_kernel" -s 4 -c 2 \
    -o $O/prof_det python bench.py --steps 3 --warmup 3 --e2e-iters 0 --no-cpu-baseline --stochastic-steps 0 \
    > $O/ncu_det.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"weighted_residual|gather_kernel" -s 6 -c 2 \
    -o $O/prof_sto python bench.py --steps 3 --warmup 3 --e2e-iters 0 --no-cpu-baseline --stochastic-steps 3 \
    > $O/ncu_sto.log 2>&1
ls -la $O
