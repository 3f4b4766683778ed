#!/bin/bash
OUT=gpurun_out/r02v; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > $OUT/tests.log 2>&1; echo "tests $?"
timeout 600 python scripts/trace_c4.py c4_road 0 > $OUT/trace_c4.txt 2>&1; echo "trace $?"
for ns in 0 128 512; do
  GR_BAR_NS=$ns timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-extras > $OUT/c2_auto_$ns.json 2>/dev/null; echo "c2 auto $ns $?"
  GR_BAR_NS=$ns timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --direction push --no-extras > $OUT/c2_push_$ns.json 2>/dev/null; echo "c2 push $ns $?"
  GR_BAR_NS=$ns timeout 600 python bench.py --config c3_orkut --steps 10 --warmup 3 --no-cpu-baseline --no-extras > $OUT/c3_bfs_$ns.json 2>/dev/null; echo "c3 bfs $ns $?"
  GR_BAR_NS=$ns timeout 900 python bench.py --config c4_road --steps 3 --warmup 3 --no-cpu-baseline --no-extras > $OUT/c4_bfs_$ns.json 2>/dev/null; echo "c4 bfs $ns $?"
  GR_BAR_NS=$ns timeout 900 python bench.py --config c4_road --prim sssp --steps 3 --warmup 3 --no-cpu-baseline --no-extras > $OUT/c4_sssp_$ns.json 2>/dev/null; echo "c4 sssp $ns $?"
done
GR_LAZY_R=0 timeout 600 python bench.py --config c3_orkut --steps 10 --warmup 3 --no-cpu-baseline --no-extras > $OUT/c3_bfs_nolazy.json 2>/dev/null; echo "c3 nolazy $?"
GR_LAZY_R=0 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --direction push --no-extras > $OUT/c2_push_nolazy.json 2>/dev/null; echo "c2 push nolazy $?"
