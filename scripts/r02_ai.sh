#!/bin/bash
for c in c2_kron21 c3_orkut c5_kron25 c1_rmat16; do
 for v in "0 0" "1 0" "2 0" "0 16" "1 16" "2 16"; do
  set -- $v
  GR_PULL_STAY=$1 GR_SPARSE_GRAB=$2 timeout 600 python bench.py --config $c --steps 16 --warmup 3 --no-cpu-baseline --no-extras 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$c stay=$1 grab=$2', round(d['ms_per_step'],4))"
 done
done
