#!/bin/bash
# A/B the stochastic-mode step under env settings: tools/ab_sto.sh "VAR=a" "VAR=b" ...
for cfg in "$@"; do
  for rep in 1 2; do
    env $cfg python bench.py --no-cpu-baseline --e2e-iters 0 --steps 20 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); s=d['stochastic']; print('$cfg', round(s['value'],1), {k: round(v,4) for k,v in s['stage_ms'].items()})"
  done
done
