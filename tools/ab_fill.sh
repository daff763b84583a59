for lib in libfvr_b200.so libfvr_b200_rf6.so libfvr_b200_rf7.so libfvr_b200_pf4.so libfvr_b200.so; do
  echo "== $lib"; FVR_LIB=$lib python tools/e2e_trace.py gpurun_out/t_$lib.txt > /dev/null 2>&1; grep -E "fill_kernel|loop kernels" gpurun_out/t_$lib.txt | cut -c1-90
  FVR_LIB=$lib python tools/e2e_gc.py 2>&1 | tail -2
done
