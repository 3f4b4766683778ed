#!/bin/bash
OUT=gpurun_out/r02q; mkdir -p $OUT
timeout 120 ./scripts/micro/latency > $OUT/latency.txt 2>&1; echo "lat $?"
for v in "libgr_b200.so 0" "libgr_b200.so 1" "libgr_head.so 1" "libgr_lb1.so 0"; do
  set -- $v
  GR_LIB=$1 GR_LAZY_R=$2 timeout 900 python bench.py --config c3_orkut --steps 10 --warmup 3 --no-cpu-baseline --no-extras > $OUT/c3_$1_$2.json 2>$OUT/c3_$1_$2.err; echo "c3 $1 $2 $?"
done
