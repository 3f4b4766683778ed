#!/bin/bash
OUT=gpurun_out/r02o; mkdir -p $OUT
timeout 600 python scripts/trace_c4.py c4_road 0 > $OUT/trace_c4.txt 2>&1; echo "trace $?"
for lib in libgr_b200.so libgr_lb1.so libgr_head.so; do
  GR_LIB=$lib timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --direction push --no-extras > $OUT/c2_push_$lib.json 2>$OUT/c2_push_$lib.err; echo "c2 push $lib $?"
  GR_LIB=$lib timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-extras > $OUT/c2_auto_$lib.json 2>$OUT/c2_auto_$lib.err; echo "c2 auto $lib $?"
done
GR_LIB=libgr_head.so timeout 900 python bench.py --config c4_road --steps 3 --warmup 3 --no-cpu-baseline --no-extras > $OUT/c4_bfs_head.json 2>$OUT/c4_bfs_head.err; echo "c4 head $?"
