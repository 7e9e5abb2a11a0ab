# unroll variants (B2DWT_LIB=...): C3 graph with and without the fused pair
for v in "" u2 u4; do
  lib=$PWD/paper_1705_08266_b200/libb2dwt${v:+_$v}.so
  B2DWT_LIB=$lib B2DWT_F2_STATIC_FRAC=768 B2DWT_F2_TAIL_ROWS=32 python tools/fused_perf.py 2>&1 | head -2 | sed "s/^/[${v:-base}] /"
done
B2DWT_LIB=$PWD/paper_1705_08266_b200/libb2dwt_u2.so python -m pytest tests/test_gpu_fused2.py -x -q 2>&1 | tail -1
