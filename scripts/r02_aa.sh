#!/bin/bash
OUT=gpurun_out/r02aa; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > $OUT/tests.log 2>&1; echo "tests $?"
timeout 900 python -m pytest tests/test_gpu_configs.py -x -q -k c4 > $OUT/tests_c4.log 2>&1; echo "tests c4 $?"
for cl in 1 0; do
  GR_ELL_CLUSTER=$cl timeout 900 python bench.py --config c4_road --prim sssp --steps 3 --warmup 3 --no-cpu-baseline --no-extras > $OUT/c4_sssp_cl$cl.json 2>$OUT/c4_sssp_cl$cl.err; echo "c4 sssp cl=$cl $?"
done
timeout 300 python scripts/level_hist.py c4_road sssp > $OUT/hist_sssp.txt 2>&1
