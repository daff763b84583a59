mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:gather_kernel<\(bool\)0, \(int\)1, \(bool\)1, \(bool\)0>' -s 2 -c 1 -o gpurun_out/prof_stog python bench.py --steps 3 --warmup 3 --e2e-iters 0 --no-cpu-baseline --stochastic-steps 3 > gpurun_out/ncu_stog.log 2>&1
tail -2 gpurun_out/ncu_stog.log
