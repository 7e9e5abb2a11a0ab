python -m pytest tests/test_gpu_fused2.py -q -x 2>&1 | tail -1
for e in 3 4 6 8; do echo "EDGE=$e $(B2DWT_F2_EDGE_ROWS=$e python tools/fused_perf.py 2>&1 | head -1)"; done
for e in 3 4; do B2DWT_F2_EDGE_ROWS=$e python -m pytest tests/test_gpu_fused2.py -q -x 2>&1 | tail -1; done
