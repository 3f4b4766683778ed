#!/bin/bash
for c in c2_kron21 c3_orkut c1_rmat16 c5_kron25; do
 for v in "512 16384" "0 16384" "512 4096" "512 65536" "128 16384"; do
  set -- $v
  GR_SMALL_F=$1 GR_SMALL_E=$2 timeout 600 python bench.py --config $c --steps 16 --warmup 3 --no-cpu-baseline --no-extras 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$c small_f=$1 small_e=$2', round(d['ms_per_step'],4))"
 done
done
