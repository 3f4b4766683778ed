#!/bin/bash
OUT=gpurun_out/r02g; mkdir -p $OUT
timeout 2400 python -m pytest tests -m gpu -x -q > $OUT/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -5 $OUT/gpu_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --partitioned --prim sssp --steps 4 --warmup 2 > $OUT/bench_part_sssp_c3.json 2> $OUT/bench_part_sssp_c3.err; echo "psssp rc=$?"; tail -2 $OUT/bench_part_sssp_c3.err
timeout 900 python bench.py --partitioned --steps 8 --warmup 3 > $OUT/bench_part_c5.json 2> $OUT/bench_part_c5.err; echo "pbfs rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"
