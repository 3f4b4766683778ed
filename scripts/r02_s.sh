#!/bin/bash
OUT=gpurun_out/r02s; mkdir -p $OUT
for env in "GR_LAZY_R=1" "GR_LAZY_R=0"; do
  env $env timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "random_graphs" > "$OUT/tests_$env.log" 2>&1; echo "tests $env $?"
done
