#!/bin/bash
OUT=gpurun_out/r02y; mkdir -p $OUT
for lib in libgr_b200.so libgr_q3.so libgr_q4.so; do
  GR_LIB=$lib timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-extras > $OUT/c2_auto_$lib.json 2>/dev/null; echo "c2 auto $lib $?"
  GR_LIB=$lib timeout 600 python bench.py --config c3_orkut --steps 10 --warmup 3 --no-cpu-baseline --no-extras > $OUT/c3_bfs_$lib.json 2>/dev/null; echo "c3 $lib $?"
  GR_LIB=$lib timeout 600 python bench.py --config c5_kron25 --steps 8 --warmup 3 --no-cpu-baseline --no-extras > $OUT/c5_bfs_$lib.json 2>/dev/null; echo "c5 $lib $?"
  GR_LIB=$lib timeout 600 python scripts/levels.py --config c2_kron21 --directions auto --nsrc 1 > $OUT/levels_c2_$lib.txt 2>&1
done
