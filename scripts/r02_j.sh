#!/bin/bash
OUT=gpurun_out/r02j; mkdir -p $OUT
timeout 900 python bench.py --config c4_road --steps 3 --warmup 2 --no-cpu-baseline --no-extras > $OUT/c4_bfs.json 2>/dev/null; echo c4 $?
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-extras > $OUT/c2_auto.json 2>/dev/null; echo c2 $?
timeout 1800 python scripts/ablation.py --out $OUT/ablation.json > $OUT/ablation.md 2> $OUT/ablation.err; echo abl $?
for d in auto push; do
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:bfs_kernel -s 3 -c 1 \
     -o $OUT/prof_c2_$d python bench.py --steps 2 --warmup 3 --direction $d --no-cpu-baseline --no-extras > $OUT/ncu_c2_$d.log 2>&1; echo "ncu c2 $d rc=$?"
done
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sssp_kernel -s 1 -c 1 \
   -o $OUT/prof_c3_sssp python bench.py --config c3_orkut --prim sssp --steps 1 --warmup 3 --no-cpu-baseline --no-extras > $OUT/ncu_c3_sssp.log 2>&1; echo "ncu c3 sssp rc=$?"
