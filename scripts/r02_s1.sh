#!/bin/bash
# round 2, session 1: GPU suite on the new tests + per-level traces of the headline configs
OUT=gpurun_out/r02a; mkdir -p $OUT
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv > $OUT/clk.txt
timeout 600 python scripts/levels.py --config c2_kron21 --directions auto,push --nsrc 3 > $OUT/levels_c2.txt 2>&1
timeout 600 python scripts/levels.py --config c5_kron25 --directions auto --nsrc 2 > $OUT/levels_c5.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > $OUT/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/gpu_tests.log
