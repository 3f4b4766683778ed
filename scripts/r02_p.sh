#!/bin/bash
OUT=gpurun_out/r02p; mkdir -p $OUT
timeout 600 python scripts/trace_c4.py c4_road 0 > $OUT/trace_c4.txt 2>&1; echo "trace $?"
timeout 600 python scripts/trace_c4.py c4_road 2 > $OUT/trace_c4_shrink2.txt 2>&1; echo "trace2 $?"
for v in "libgr_b200.so 1" "libgr_b200.so 0" "libgr_lb1.so 1" "libgr_head.so 1"; do
  set -- $v
  GR_LIB=$1 GR_LAZY_R=$2 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --direction push --no-extras > $OUT/c2_push_$1_$2.json 2>$OUT/c2_push_$1_$2.err; echo "c2 push $1 $2 $?"
  GR_LIB=$1 GR_LAZY_R=$2 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-extras > $OUT/c2_auto_$1_$2.json 2>$OUT/c2_auto_$1_$2.err; echo "c2 auto $1 $2 $?"
done
timeout 900 python bench.py --config c4_road --steps 3 --warmup 3 --no-cpu-baseline --no-extras > $OUT/c4_bfs.json 2>$OUT/c4_bfs.err; echo "c4 $?"
timeout 900 python bench.py --config c3_orkut --steps 10 --warmup 3 --no-cpu-baseline --no-extras > $OUT/c3_bfs.json 2>$OUT/c3_bfs.err; echo "c3 $?"
GR_LIB=libgr_head.so timeout 900 python bench.py --config c3_orkut --steps 10 --warmup 3 --no-cpu-baseline --no-extras > $OUT/c3_bfs_head.json 2>$OUT/c3_bfs_head.err; echo "c3 head $?"
