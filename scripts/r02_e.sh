#!/bin/bash
OUT=gpurun_out/r02e; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pbfs.py -x -q > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/tests.log
timeout 300 python scripts/trace_levels.py c2_kron21 0 > $OUT/trace_c2_auto.txt 2>&1
timeout 600 python scripts/levels.py --config c2_kron21 --directions auto,push --nsrc 2 > $OUT/levels_c2.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:bfs_kernel -s 3 -c 1 -o $OUT/prof_c2_auto python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras > $OUT/ncu_c2_auto.log 2>&1; echo "ncu rc=$?"
