#!/bin/bash
for c in c2_kron21 c3_orkut c5_kron25; do
 for a in 14 17 20 24; do
  GR_ALPHA=$a timeout 600 python bench.py --config $c --steps 16 --warmup 3 --no-cpu-baseline --no-extras 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$c alpha=$a', round(d['ms_per_step'],4))"
 done
done
