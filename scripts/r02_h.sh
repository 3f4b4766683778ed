#!/bin/bash
OUT=gpurun_out/r02h; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_sssp_pull.py tests/test_gpu_bc.py tests/test_gpu_parity.py -x -q > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -15 $OUT/tests.log
for d in push pull auto; do
  timeout 600 python bench.py --config c3_orkut --prim sssp --steps 4 --warmup 2 --no-cpu-baseline --no-extras --sssp-direction $d > $OUT/bench_c3_sssp_$d.json 2> $OUT/bench_c3_sssp_$d.err; echo "c3 sssp $d rc=$?"
done
for d in push auto; do
  timeout 900 python bench.py --config c4_road --prim sssp --steps 2 --warmup 1 --no-cpu-baseline --no-extras --sssp-direction $d > $OUT/bench_c4_sssp_$d.json 2> $OUT/bench_c4_sssp_$d.err; echo "c4 sssp $d rc=$?"
done
for d in push auto; do
  timeout 600 python bench.py --prim bc --steps 4 --warmup 2 --no-cpu-baseline --bc-direction $d > $OUT/bench_c2_bc_$d.json 2> $OUT/bench_c2_bc_$d.err; echo "c2 bc $d rc=$?"
  timeout 600 python bench.py --config c3_orkut --prim bc --steps 4 --warmup 2 --no-cpu-baseline --bc-direction $d > $OUT/bench_c3_bc_$d.json 2> $OUT/bench_c3_bc_$d.err; echo "c3 bc $d rc=$?"
done
timeout 600 python scripts/levels.py --config c3_orkut --prim sssp --nsrc 1 --maxrows 60 > $OUT/levels_c3_sssp.txt 2>&1
