#!/bin/bash
OUT=gpurun_out/r02h; mkdir -p $OUT
timeout 2400 python -m pytest tests/ -m gpu -x -q > $OUT/gpu_tests.log 2>&1; echo "tests $?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke $?"
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench $?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref $?"
bash scripts/gpu_measure.sh r02h bench
timeout 600 python bench.py --partitioned --steps 8 --no-extras > $OUT/bench_c5_part.json 2>/dev/null; echo "part $?"
timeout 1800 python scripts/ablation.py --out $OUT/ablation.json > $OUT/ablation.md 2> $OUT/ablation.err; echo "abl $?"
