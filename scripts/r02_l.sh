#!/bin/bash
# Bounded-degree (ELL) adjacency: parity + C4 BFS/SSSP with and without it
OUT=gpurun_out/r02l; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "bounded or closed_form or random_graphs or strategies or long_path" > $OUT/tests.log 2>&1; echo "tests $?"
timeout 900 python -m pytest tests/test_gpu_sssp_pull.py tests/test_gpu_sanitizer.py -x -q > $OUT/tests_pull.log 2>&1; echo "tests pull $?"
for ell in 1 0; do
  GR_ELL=$ell timeout 900 python bench.py --config c4_road --steps 3 --warmup 3 --no-cpu-baseline --no-extras > $OUT/c4_bfs_ell$ell.json 2>$OUT/c4_bfs_ell$ell.err; echo "c4 bfs ell=$ell $?"
  GR_ELL=$ell timeout 900 python bench.py --config c4_road --prim sssp --steps 3 --warmup 3 --no-cpu-baseline --no-extras > $OUT/c4_sssp_ell$ell.json 2>$OUT/c4_sssp_ell$ell.err; echo "c4 sssp ell=$ell $?"
done
timeout 900 python -m pytest tests/test_gpu_configs.py -x -q -k c4 > $OUT/tests_c4.log 2>&1; echo "tests c4 $?"
# source-level profile of the headline (C2 push-pull) kernel
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:bfs_kernel -s 3 -c 1 \
   -o $OUT/prof_c2_auto python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras > $OUT/ncu_c2_auto.log 2>&1; echo "ncu c2 auto $?"
ncu -i $OUT/prof_c2_auto.ncu-rep --page source --csv --print-source cuda > $OUT/src_c2_auto_cuda.csv 2>$OUT/src.err; echo "src $?"
ncu -i $OUT/prof_c2_auto.ncu-rep --page source --csv --print-source sass > $OUT/src_c2_auto_sass.csv 2>>$OUT/src.err
ncu -i $OUT/prof_c2_auto.ncu-rep --page raw --csv > $OUT/raw_c2_auto.csv 2>/dev/null
