#!/bin/bash
# A/B experiment builds of the library (csrc/Makefile OUT=...):
#   tools/ab_lib.sh libfvr_b200.so "libfvr_b200_x.so FVR_X=1" ...
# (extra words of an argument are environment settings for that build);
# prints the device-timed step, stage times and the public-API e2e of each
for spec in "$@"; do
  set -- $spec
  lib=$1; shift
  for rep in 1 2; do
    env FVR_LIB=$lib "$@" python bench.py --no-cpu-baseline --steps 50 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$spec', round(d['value'],1), {k: round(v,4) for k,v in d['stage_ms'].items()}, 'sto', round(d['stochastic']['value'],1), {k: round(v,4) for k,v in d['stochastic']['stage_ms'].items()}, 'e2e', round(d['e2e']['value'],1), [round(x,2) for x in d['e2e']['calls_ms']])"
  done
done
