for r in 0 2 3 4; do echo "RAMP=$r"; B2DWT_PIPE_RAMP=$r BANDS="12 16 24" python tools/e2e_probe.py 2>&1 | grep -v idwt | tail -4; done
python -m pytest tests/test_gpu_parity.py -q -k "host" 2>&1 | tail -1
