#!/bin/bash
OUT=gpurun_out/r02x; mkdir -p $OUT
for mp in 0 128 512 2048; do
  GR_LB_MIN_PIECE=$mp timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-extras > $OUT/c2_auto_$mp.json 2>/dev/null; echo "c2 auto $mp $?"
  GR_LB_MIN_PIECE=$mp timeout 600 python bench.py --config c3_orkut --steps 10 --warmup 3 --no-cpu-baseline --no-extras > $OUT/c3_bfs_$mp.json 2>/dev/null; echo "c3 $mp $?"
  GR_LB_MIN_PIECE=$mp timeout 600 python bench.py --config c5_kron25 --steps 8 --warmup 3 --no-cpu-baseline --no-extras > $OUT/c5_bfs_$mp.json 2>/dev/null; echo "c5 $mp $?"
done
timeout 600 python scripts/levels.py --config c2_kron21 --directions auto --nsrc 2 > $OUT/levels_c2.txt 2>&1
GR_LB_MIN_PIECE=512 timeout 600 python scripts/levels.py --config c2_kron21 --directions auto --nsrc 2 > $OUT/levels_c2_512.txt 2>&1
