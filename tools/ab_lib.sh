# A/B/C of the C3 pyramid between the default library and experiment builds:
#   LIBS="paper_1705_08266_b200/libb2dwt_X.so ..." MODES=1:1,0:1 bash tools/ab_lib.sh
for rep in 1 2 3; do
  echo "default $(MODES=${MODES:-1:1} python tools/fused_perf.py 2>&1 | tr '\n' ' ')"
  for l in $LIBS; do
    echo "$(basename $l) $(B2DWT_LIB=$PWD/$l MODES=${MODES:-1:1} python tools/fused_perf.py 2>&1 | tr '\n' ' ')"
  done
done
