mkdir -p gpurun_out
for r in 1 2; do for s in 1 0; do
FVR_PAD_ZERO=$s python bench.py --no-cpu-baseline --stochastic-steps 0 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('pad_zero=$s', round(d['value'],1), round(d['e2e']['value'],1), sorted(round(x,2) for x in d['e2e']['calls_ms']))" >> gpurun_out/ab_pz_bench.txt
done; done
