#!/bin/bash
OUT=gpurun_out/r02ag; mkdir -p $OUT
for lib in libgr_b200.so libgr_noagg.so; do
 for r in 1 2; do
  GR_LIB=$lib timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-extras > $OUT/c2_${lib}_$r.json 2>/dev/null; echo "c2 $lib $?"
 done
  GR_LIB=$lib timeout 600 python bench.py --config c3_orkut --steps 10 --warmup 3 --no-cpu-baseline --no-extras > $OUT/c3_$lib.json 2>/dev/null; echo "c3 $lib $?"
  GR_LIB=$lib timeout 600 python bench.py --config c5_kron25 --steps 8 --warmup 3 --no-cpu-baseline --no-extras > $OUT/c5_$lib.json 2>/dev/null; echo "c5 $lib $?"
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "random or mid_size or c1 or strategies or golden" > $OUT/tests.log 2>&1; echo "tests $?"
