#!/bin/bash
OUT=gpurun_out/r02ae; mkdir -p $OUT
for d in 1024 2048 4096 8192 16384 65536 4294967295; do
  timeout 900 python bench.py --config c4_road --prim sssp --delta $d --steps 3 --warmup 2 --no-cpu-baseline --no-extras > $OUT/c4_sssp_d$d.json 2>/dev/null; echo "d=$d $?"
done
for d in 2 3 4 6; do
  timeout 900 python bench.py --config c3_orkut --prim sssp --delta $d --steps 4 --warmup 2 --no-cpu-baseline --no-extras > $OUT/c3_sssp_d$d.json 2>/dev/null; echo "c3 d=$d $?"
done
