# fused kernel work split: tests, then C3 graph time vs static fraction / tail chunk
# (MODES picks fast:fuse pairs of tools/fused_perf.py; SFS / TRS the sweep values)
[ -n "$NOTEST" ] || python -m pytest tests/test_gpu_fused2.py tests/test_gpu_guard.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -1
for rep in 1 2; do for sf in ${SFS:-640 704 768 832 896}; do for tr in ${TRS:-16}; do
  echo "F2SF=$sf TR=$tr $(B2DWT_F2_STATIC_FRAC=$sf B2DWT_F2_TAIL_ROWS=$tr MODES=${MODES:-1:1} python tools/fused_perf.py 2>&1 | sed -n 1p)"
done; done; done
