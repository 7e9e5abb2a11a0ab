# fused kernel guided claim size remaining / (k x CTAs) x static share x min chunk (C3 levels 0+1)
for rep in 1 2; do for k in ${KS:-1}; do for sf in ${SFS:-768 832 896 960}; do for tr in ${TRS:-8 12 16 24}; do
  echo "K=$k SF=$sf TR=$tr $(B2DWT_F2_GUIDED=$k B2DWT_F2_STATIC_FRAC=$sf B2DWT_F2_TAIL_ROWS=$tr MODES=1:1 python tools/fused_perf.py 2>&1 | sed -n 1p)"
done; done; done; done
