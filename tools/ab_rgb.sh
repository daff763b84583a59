for lib in libfvr_b200.so libfvr_b200_g3a.so libfvr_b200_g3b.so libfvr_b200_g3c.so libfvr_b200.so; do
  FVR_LIB=$lib python tools/rgb_bench.py 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', {k: round(v['rgb_iters_per_s'],1) for k,v in d.items() if isinstance(v, dict)})"
done
