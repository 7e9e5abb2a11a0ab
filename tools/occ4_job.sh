export PROGRAMS=cdf97/separable-convolution
for rep in 1 2; do
  echo "default $(python tools/program_perf.py 2>&1 | tr '\n' ' ')"
  echo "occ4 $(B2DWT_LIB=$PWD/paper_1705_08266_b200/libb2dwt_occ4.so python tools/program_perf.py 2>&1 | tr '\n' ' ')"
done
unset PROGRAMS
python tools/scheme_pyramid.py
