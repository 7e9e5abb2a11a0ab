# levels 2+3 fused launch (C3): CTA count (B2DWT_F2_MIN_ROWS) and dynamic tail for small launches (B2DWT_F2_DYN_MIN)
for rep in 1 2; do for mr in 8 16 24 32 48; do for dm in 64 16; do
  echo "MR=$mr DM=$dm $(B2DWT_F2_MIN_ROWS=$mr B2DWT_F2_DYN_MIN=$dm MODES=1:1 python tools/fused_perf.py 2>&1 | sed -n 1p)"
done; done; done
