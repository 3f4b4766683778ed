#!/bin/bash
# C4 level timeline (trace build) + C4/C2 bench with ELL + lazy R + dual search
OUT=gpurun_out/r02m; mkdir -p $OUT
timeout 600 python scripts/trace_c4.py c4_road 0 > $OUT/trace_c4.txt 2>&1; echo "trace $?"
timeout 600 python scripts/trace_levels.py c2_kron21 0 > $OUT/trace_c2.txt 2>&1; echo "trace c2 $?"
timeout 900 python bench.py --config c4_road --steps 3 --warmup 3 --no-cpu-baseline --no-extras > $OUT/c4_bfs.json 2>$OUT/c4_bfs.err; echo "c4 bfs $?"
timeout 900 python bench.py --config c4_road --prim sssp --steps 3 --warmup 3 --no-cpu-baseline --no-extras > $OUT/c4_sssp.json 2>$OUT/c4_sssp.err; echo "c4 sssp $?"
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $OUT/c2.json 2>$OUT/c2.err; echo "c2 $?"
GR_LAZY_R=0 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $OUT/c2_nolazy.json 2>$OUT/c2_nolazy.err; echo "c2 nolazy $?"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > $OUT/tests.log 2>&1; echo "tests $?"
