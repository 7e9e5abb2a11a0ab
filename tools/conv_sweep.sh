P="cdf97/separable-convolution,cdf97/separable-lifting,cdf97/non-separable-split"
ARITH=fast PROGRAMS=$P python tools/program_perf.py | sed 's/^/[base] /'
ARITH=fast PROGRAMS=cdf97/separable-convolution B2DWT_STATIC_FRAC=1024 python tools/program_perf.py | sed 's/^/[static1024] /'
ARITH=fast PROGRAMS=cdf97/separable-convolution B2DWT_TAIL_ROWS=64 python tools/program_perf.py | sed 's/^/[tail64] /'
python tools/fused_perf.py 2>&1 | head -2
python -m pytest tests/test_gpu_fused2.py tests/test_gpu_parity.py tests/test_gpu_parity_c2.py -q -x 2>&1 | tail -1
