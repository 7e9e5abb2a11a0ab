for e in 4 8; do for p in "0,2" "0,3"; do
  echo "EDGE=$e PAIRS=$p $(B2DWT_F2_EDGE_ROWS=$e B2DWT_FUSE2_PAIRS=$p python tools/fused_perf.py 2>&1 | head -1)"
done; done
