#!/bin/bash
OUT=gpurun_out/r02i; mkdir -p $OUT
for lib in libgr_b200.so libgr_b200_nospec.so; do
  GR_LIB=$lib timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-extras > $OUT/c2_auto_$lib.json 2>/dev/null
  GR_LIB=$lib timeout 600 python bench.py --steps 8 --warmup 3 --direction push --no-cpu-baseline --no-extras > $OUT/c2_push_$lib.json 2>/dev/null
  GR_LIB=$lib timeout 900 python bench.py --config c4_road --steps 3 --warmup 2 --no-cpu-baseline --no-extras > $OUT/c4_bfs_$lib.json 2>/dev/null
  GR_LIB=$lib timeout 900 python bench.py --config c3_orkut --steps 8 --warmup 3 --no-cpu-baseline --no-extras > $OUT/c3_bfs_$lib.json 2>/dev/null
done
timeout 600 python scripts/trace_levels.py c4_road 0 > $OUT/trace_c4.txt 2>&1
timeout 600 python scripts/levels.py --config c4_road --directions auto --nsrc 1 --maxrows 30 > $OUT/levels_c4.txt 2>&1
