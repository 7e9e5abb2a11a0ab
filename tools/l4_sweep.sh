# C3 level 4 (1024^2 input): tile kernel window rows 16 / 32 vs the stream kernel (TILE_MAX_QUADS=0)
for rep in 1 2; do
  for v in "B2DWT_TILE_ROWS=16" "B2DWT_TILE_ROWS=32" "B2DWT_TILE_MAX_QUADS=0" "B2DWT_TILE_MAX_QUADS=0 B2DWT_MIN_ROWS=8" "B2DWT_TILE_MAX_QUADS=0 B2DWT_MIN_ROWS=4"; do
    echo "$v $(env $v MODES=1:1 python tools/fused_perf.py 2>&1 | sed -n 1p)"
  done
done
