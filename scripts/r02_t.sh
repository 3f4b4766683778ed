#!/bin/bash
OUT=gpurun_out/r02t; mkdir -p $OUT
GR_LAZY_R=0 timeout 300 python scripts/debug_sssp.py > $OUT/debug_nolazy.txt 2>&1; echo "dbg0 $?"
timeout 300 python scripts/debug_sssp.py > $OUT/debug.txt 2>&1; echo "dbg1 $?"
timeout 2400 python -m pytest tests/ -m gpu -x -q > $OUT/tests.log 2>&1; echo "tests $?"
