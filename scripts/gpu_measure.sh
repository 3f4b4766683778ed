#!/bin/bash
# One GPU session: bench lines, full-size parity, ncu launch list + full capture.
# Usage (under gpurun): bash scripts/gpu_measure.sh <tag> [what...]
# what: bench, configs, launches, ncu, sssp   (default: all)
set -u
TAG=${1:-r01}; shift || true
WHAT=${*:-"bench configs launches ncu sssp"}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi -q -d CLOCK > $OUT/clocks_start.txt 2>&1
for w in $WHAT; do
case $w in
bench)
  timeout 900 python bench.py > $OUT/bench_c2_auto.json 2> $OUT/bench_c2_auto.err; echo "bench rc=$?"
  timeout 900 python bench.py --direction push --no-extras > $OUT/bench_c2_push.json 2> $OUT/bench_c2_push.err; echo "bench push rc=$?"
  ;;
sssp)
  timeout 900 python bench.py --config c3_orkut --prim sssp --steps 4 --no-extras > $OUT/bench_c3_sssp.json 2> $OUT/bench_c3_sssp.err; echo "bench c3 sssp rc=$?"
  timeout 900 python bench.py --config c3_orkut --prim bfs --steps 8 --no-extras > $OUT/bench_c3_bfs.json 2> $OUT/bench_c3_bfs.err; echo "bench c3 bfs rc=$?"
  timeout 900 python bench.py --config c4_road --prim bfs --steps 4 --no-extras > $OUT/bench_c4_bfs.json 2> $OUT/bench_c4_bfs.err; echo "bench c4 bfs rc=$?"
  timeout 900 python bench.py --config c4_road --prim sssp --steps 2 --no-extras > $OUT/bench_c4_sssp.json 2> $OUT/bench_c4_sssp.err; echo "bench c4 sssp rc=$?"
  ;;
configs)
  timeout 1500 python -m pytest tests -m "gpu and slow" -x -q > $OUT/configs_tests.log 2>&1; echo "configs rc=$?"; tail -5 $OUT/configs_tests.log
  ;;
launches)
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
     python bench.py --steps 4 --warmup 1 --no-cpu-baseline --no-extras > $OUT/launches_bench.json 2>&1; echo "launches rc=$?"
  ;;
ncu)
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:bfs_kernel -s 2 -c 1 \
     -o $OUT/prof_bfs_push python bench.py --steps 2 --warmup 1 --direction push --no-cpu-baseline --no-extras > $OUT/ncu_push.log 2>&1; echo "ncu push rc=$?"
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:bfs_kernel -s 2 -c 1 \
     -o $OUT/prof_bfs_auto python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-extras > $OUT/ncu_auto.log 2>&1; echo "ncu auto rc=$?"
  ;;
esac
done
for f in $OUT/*.json; do echo "== $f"; head -c 1500 $f; echo; done
