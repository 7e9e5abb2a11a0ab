# fused kernel TMA L2 promotion (bytes) on C3, final work split
for rep in 1 2; do for p in 0 64 128 256; do
  echo "PROMO=$p $(B2DWT_F2_L2PROMO=$p MODES=1:1 python tools/fused_perf.py 2>&1 | sed -n 1p)"
done; done
