#!/bin/bash
OUT=gpurun_out/r02d; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_pbfs.py -x -q > $OUT/pbfs_tests.log 2>&1; echo "pbfs tests rc=$?"; tail -3 $OUT/pbfs_tests.log
timeout 300 python scripts/balance.py c2_kron21 auto > $OUT/balance_c2_auto.txt 2>&1
timeout 300 python scripts/trace_levels.py c2_kron21 0 > $OUT/trace_c2_auto.txt 2>&1
timeout 900 python bench.py --partitioned --steps 8 --warmup 3 > $OUT/bench_part_c5.json 2> $OUT/bench_part_c5.err; echo "part bench rc=$?"; tail -3 $OUT/bench_part_c5.err
