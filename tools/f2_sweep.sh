for rep in 1 2; do
  python tools/fused_perf.py 2>&1 | head -1 | sed "s/^/[hints] /"
  B2DWT_LIB=$PWD/paper_1705_08266_b200/libb2dwt_nohint.so python tools/fused_perf.py 2>&1 | head -1 | sed "s/^/[nohint] /"
done
for pr in 256 64; do for c in c4 c5; do echo "$c L2PROMO=$pr $(B2DWT_L2PROMO=$pr python bench.py --config $c --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d[\"value\"],1), round(d[\"ms_per_step\"],3))")"; done; done
for pr in 256 64; do echo "stream L0 only L2PROMO=$pr $(B2DWT_L2PROMO=$pr python tools/fused_perf.py 2>&1 | sed -n 2p)"; done
python -m pytest tests/test_gpu_fused2.py -q -x 2>&1 | tail -1
