python -m pytest tests/test_gpu_fused2.py tests/test_gpu_guard.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -1
for rep in 1 2; do for sf in 704 768 832; do for tr in 8 16 32; do
  echo "F2SF=$sf TR=$tr $(B2DWT_F2_STATIC_FRAC=$sf B2DWT_F2_TAIL_ROWS=$tr python tools/fused_perf.py 2>&1 | sed -n 1p)"
done; done; done
python tools/fused_perf.py 2>&1 | sed -n 3p
