#!/bin/bash
OUT=gpurun_out/r02n; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > $OUT/tests.log 2>&1; echo "tests $?"
timeout 600 python scripts/trace_c4.py c4_road 0 > $OUT/trace_c4.txt 2>&1; echo "trace $?"
timeout 900 python bench.py --config c4_road --steps 3 --warmup 3 --no-cpu-baseline --no-extras > $OUT/c4_bfs.json 2>$OUT/c4_bfs.err; echo "c4 bfs $?"
timeout 900 python bench.py --config c4_road --prim sssp --steps 3 --warmup 3 --no-cpu-baseline --no-extras > $OUT/c4_sssp.json 2>$OUT/c4_sssp.err; echo "c4 sssp $?"
