#!/bin/bash
OUT=gpurun_out/r02j2; mkdir -p $OUT
timeout 2400 python -m pytest tests/ -m gpu -x -q > $OUT/gpu_tests.log 2>&1; echo "tests $?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke $?"
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench $?"
timeout 900 python bench.py --config c4_road --prim sssp --steps 3 --warmup 2 --no-extras > $OUT/bench_c4_sssp.json 2>/dev/null; echo "c4 sssp $?"
timeout 900 python bench.py --config c1_rmat16 --no-extras > $OUT/bench_c1.json 2>/dev/null; echo "c1 $?"
