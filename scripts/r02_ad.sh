#!/bin/bash
OUT=gpurun_out/r02ad; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sssp_pull.py -x -q > $OUT/tests.log 2>&1; echo "tests $?"
for lib in libgr_b200.so libgr_prev.so; do
  GR_LIB=$lib timeout 600 python bench.py --config c3_orkut --prim sssp --steps 5 --warmup 3 --no-cpu-baseline --no-extras > $OUT/c3_sssp_$lib.json 2>/dev/null; echo "c3 sssp $lib $?"
done
