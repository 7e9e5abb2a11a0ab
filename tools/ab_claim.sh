export PROGRAMS=cdf97/separable-convolution,cdf97/non-separable-split,cdf97/separable-lifting
for rep in 1 2; do
 for lib in default cta; do
  if [ $lib = default ]; then unset B2DWT_LIB; else export B2DWT_LIB=$PWD/paper_1705_08266_b200/libb2dwt_cta.so; fi
  python tools/program_perf.py 2>&1 | sed "s/^/$lib /"
 done
done
