# fused static share 768 vs 832 (final kernel), both arithmetic modes, same box
for rep in 1 2 3; do for sf in 768 832; do
  echo "SF=$sf $(B2DWT_F2_STATIC_FRAC=$sf MODES=1:1,0:1 python tools/fused_perf.py 2>&1 | sed 's/fuse=True: graph//; s/| groups[^f]*//g' | tr '\n' ' ')"
done; done
