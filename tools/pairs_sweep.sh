# C3: which levels start a fused pair (B2DWT_FUSE2_PAIRS) with the final fused kernel
for rep in 1 2; do for p in "0,2" "0,3" "0"; do
  echo "PAIRS=$p $(B2DWT_FUSE2_PAIRS=$p B2DWT_FUSE2_MIN_QUADS=1 MODES=1:1 python tools/fused_perf.py 2>&1 | sed -n 1p)"
done; done
