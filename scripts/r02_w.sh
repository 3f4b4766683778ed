#!/bin/bash
OUT=gpurun_out/r02w; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > $OUT/tests.log 2>&1; echo "tests $?"
timeout 900 python -m pytest tests/test_gpu_configs.py -x -q -k c4 > $OUT/tests_c4.log 2>&1; echo "tests c4 $?"
for cl in 1 0; do
  GR_ELL_CLUSTER=$cl timeout 900 python bench.py --config c4_road --steps 3 --warmup 3 --no-cpu-baseline --no-extras > $OUT/c4_bfs_cl$cl.json 2>$OUT/c4_bfs_cl$cl.err; echo "c4 bfs cl=$cl $?"
done
GR_ELL_CLUSTER_SIZE=8 timeout 900 python bench.py --config c4_road --steps 3 --warmup 3 --no-cpu-baseline --no-extras > $OUT/c4_bfs_cl8.json 2>$OUT/c4_bfs_cl8.err; echo "c4 bfs cl8 $?"
