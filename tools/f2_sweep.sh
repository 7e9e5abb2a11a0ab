python -m pytest tests/test_gpu_fused2.py -q -x 2>&1 | tail -1
for mb in 268435456 536870912 1073741824 2147483648; do
  echo "MAXLAUNCH=$mb $(B2DWT_MAX_LAUNCH_BYTES=$mb python tools/fused_perf.py 2>&1 | head -1)"
done
