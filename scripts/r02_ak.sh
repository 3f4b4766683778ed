#!/bin/bash
for c in c2_kron21 c3_orkut c5_kron25 c1_rmat16; do
 for v in "14 24" "6 24" "10 24" "20 24" "30 24" "14 8" "14 64" "14 200"; do
  set -- $v
  GR_ALPHA=$1 GR_BETA=$2 timeout 600 python bench.py --config $c --steps 16 --warmup 3 --no-cpu-baseline --no-extras 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$c alpha=$1 beta=$2', round(d['ms_per_step'],4), d['levels_per_step'])"
 done
done
