#!/bin/bash
OUT=gpurun_out/r02c; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_pbfs.py -x -q > $OUT/pbfs_tests.log 2>&1; echo "pbfs tests rc=$?"; tail -30 $OUT/pbfs_tests.log
timeout 600 python scripts/levels.py --config c2_kron21 --directions auto --nsrc 3 > $OUT/levels_c2.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > $OUT/parity_tests.log 2>&1; echo "parity rc=$?"; tail -3 $OUT/parity_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
