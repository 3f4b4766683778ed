#!/bin/bash
OUT=gpurun_out/r02ab; mkdir -p $OUT
timeout 900 python bench.py --config c4_road --prim sssp --steps 3 --warmup 3 --no-cpu-baseline --no-extras > $OUT/c4_sssp.json 2>$OUT/c4_sssp.err; echo "c4 sssp $?"
timeout 900 python bench.py --config c4_road --steps 3 --warmup 3 --no-cpu-baseline --no-extras > $OUT/c4_bfs.json 2>$OUT/c4_bfs.err; echo "c4 bfs $?"
timeout 2400 python -m pytest tests/ -m gpu -x -q > $OUT/tests.log 2>&1; echo "tests $?"
