#!/bin/bash
OUT=gpurun_out/r02u; mkdir -p $OUT
timeout 600 python scripts/trace_c4.py c4_road 0 > $OUT/trace_c4.txt 2>&1; echo "trace $?"
timeout 600 python scripts/trace_levels.py c2_kron21 0 > $OUT/trace_c2.txt 2>&1; echo "trace c2 $?"
for lib in libgr_b200.so libgr_head.so; do
  GR_LIB=$lib timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-extras > $OUT/c2_auto_$lib.json 2>/dev/null; echo "c2 auto $lib $?"
  GR_LIB=$lib timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --direction push --no-extras > $OUT/c2_push_$lib.json 2>/dev/null; echo "c2 push $lib $?"
  GR_LIB=$lib timeout 600 python bench.py --config c3_orkut --steps 10 --warmup 3 --no-cpu-baseline --no-extras > $OUT/c3_bfs_$lib.json 2>/dev/null; echo "c3 bfs $lib $?"
  GR_LIB=$lib timeout 600 python bench.py --config c3_orkut --prim sssp --steps 4 --warmup 3 --no-cpu-baseline --no-extras > $OUT/c3_sssp_$lib.json 2>/dev/null; echo "c3 sssp $lib $?"
  GR_LIB=$lib timeout 900 python bench.py --config c4_road --steps 3 --warmup 3 --no-cpu-baseline --no-extras > $OUT/c4_bfs_$lib.json 2>/dev/null; echo "c4 bfs $lib $?"
  GR_LIB=$lib timeout 900 python bench.py --config c4_road --prim sssp --steps 3 --warmup 3 --no-cpu-baseline --no-extras > $OUT/c4_sssp_$lib.json 2>/dev/null; echo "c4 sssp $lib $?"
  GR_LIB=$lib timeout 900 python bench.py --config c5_kron25 --steps 8 --warmup 3 --no-cpu-baseline --no-extras > $OUT/c5_bfs_$lib.json 2>/dev/null; echo "c5 $lib $?"
  GR_LIB=$lib timeout 900 python bench.py --partitioned --steps 8 --warmup 3 --no-cpu-baseline --no-extras > $OUT/c5_part_$lib.json 2>/dev/null; echo "c5 part $lib $?"
  GR_LIB=$lib timeout 900 python bench.py --config c2_kron21 --prim bc --steps 5 --warmup 3 --no-cpu-baseline --no-extras > $OUT/c2_bc_$lib.json 2>/dev/null; echo "c2 bc $lib $?"
done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pbfs.py tests/test_gpu_bc.py -x -q > $OUT/tests.log 2>&1; echo "tests $?"
