for p in 0 1; do
  for c in c4 c5; do echo "PACK=$p $c $(B2DWT_STRIP_PACK=$p python bench.py --config $c --steps 10 --warmup 3 --no-scale-configs 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d[\"value\"],1), round(d[\"ms_per_step\"],3))")"; done
  echo "PACK=$p $(B2DWT_STRIP_PACK=$p python tools/fused_perf.py 2>&1 | sed -n 2p)"
  B2DWT_STRIP_PACK=$p ARITH=fast PROGRAMS=cdf97/non-separable-split,cdf53/non-separable-split,cdf97/separable-convolution python tools/program_perf.py | sed "s/^/PACK=$p /"
done
B2DWT_STRIP_PACK=1 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_c2.py tests/test_gpu_fuzz.py tests/test_gpu_guard.py -q -x 2>&1 | tail -1
