#!/bin/bash
# A/B a bench stage time under env settings: tools/ab_env.sh "VAR=a" "VAR=b" ...
for cfg in "$@"; do
  for rep in 1 2; do
    env $cfg python bench.py --no-cpu-baseline --e2e-iters 0 --steps 50 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', round(d['value'],1), {k: round(v,4) for k,v in d['stage_ms'].items()})"
  done
done
