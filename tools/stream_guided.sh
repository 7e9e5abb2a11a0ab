# stream kernel (C4 batch, C5 row strips): guided tail claims remaining / (k x CTAs), k = 0 (fixed chunks) .. 2
for rep in 1 2; do for k in 0 1 2; do for c in c4 c5; do
  echo "K=$k $c $(B2DWT_GUIDED=$k python bench.py --config $c --no-cpu --steps 10 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"],1), round(d["ms_per_step"],3))')"
done; done; done
