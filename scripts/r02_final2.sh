#!/bin/bash
OUT=gpurun_out/r02g; mkdir -p $OUT
timeout 2400 python -m pytest tests/ -m gpu -x -q > $OUT/gpu_tests.log 2>&1; echo "tests $?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke $?"
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench $?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref $?"
