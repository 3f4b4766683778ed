#!/bin/bash
OUT=gpurun_out/r02ac; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > $OUT/tests.log 2>&1; echo "tests $?"
for lib in libgr_b200.so libgr_prev.so; do
 for rep in 1 2; do
  GR_LIB=$lib timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-extras > $OUT/c2_auto_${lib}_$rep.json 2>/dev/null; echo "c2 $lib $?"
 done
  GR_LIB=$lib timeout 600 python bench.py --config c3_orkut --steps 10 --warmup 3 --no-cpu-baseline --no-extras > $OUT/c3_bfs_$lib.json 2>/dev/null; echo "c3 $lib $?"
  GR_LIB=$lib timeout 600 python bench.py --config c1_rmat16 --steps 10 --warmup 3 --no-cpu-baseline --no-extras > $OUT/c1_$lib.json 2>/dev/null; echo "c1 $lib $?"
  GR_LIB=$lib timeout 600 python bench.py --config c5_kron25 --steps 8 --warmup 3 --no-cpu-baseline --no-extras > $OUT/c5_$lib.json 2>/dev/null; echo "c5 $lib $?"
  GR_LIB=$lib timeout 600 python bench.py --steps 10 --warmup 3 --direction push --no-cpu-baseline --no-extras > $OUT/c2_push_$lib.json 2>/dev/null; echo "c2 push $lib $?"
done
