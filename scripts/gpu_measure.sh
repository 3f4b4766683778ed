#!/bin/bash
# One GPU session: bench lines for every config, ncu launch list and full
# captures of the top kernel, summaries. Usage (under gpurun):
#   bash scripts/gpu_measure.sh <tag> [what...]
# what: bench, configs, launches, ncu   (default: bench launches ncu)
set -u
TAG=${1:-r01}; shift || true
WHAT=${*:-"bench launches ncu"}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi -q -d CLOCK > $OUT/clocks_start.txt 2>&1
b() {  # name, bench args...
  local name=$1; shift
  timeout 900 python bench.py "$@" > $OUT/bench_$name.json 2> $OUT/bench_$name.err; echo "bench $name rc=$?"
}
for w in $WHAT; do
case $w in
bench)
  b c2_auto
  b c2_push --direction push --no-extras
  b c1 --config c1_rmat16 --no-extras
  b c3_bfs --config c3_orkut --prim bfs --no-extras
  b c3_sssp --config c3_orkut --prim sssp --steps 4 --no-extras
  b c4_bfs --config c4_road --prim bfs --steps 4 --no-extras
  b c4_sssp --config c4_road --prim sssp --steps 2 --no-extras
  b c5 --config c5_kron25 --steps 8 --no-extras --cpu-sample-s 10
  ;;
more)
  b c5_part --partitioned --steps 8 --no-extras
  b c3_part_sssp --partitioned --config c3_orkut --prim sssp --steps 4 --no-extras
  b c2_bc --prim bc --steps 5 --no-extras
  b c2_cc --prim cc --steps 5 --no-extras
  b c2_pr --prim pr --steps 3 --no-extras
  timeout 600 python scripts/level_hist.py c4_road bfs > $OUT/level_hist_c4_bfs.txt 2>&1
  timeout 600 python scripts/level_hist.py c4_road sssp > $OUT/level_hist_c4_sssp.txt 2>&1
  timeout 600 python scripts/levels.py --config c2_kron21 --directions auto,push --nsrc 2 > $OUT/levels_c2.txt 2>&1
  ;;
ncu_c4)
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:bfs_ell_cluster_kernel -s 1 -c 1 \
     -o $OUT/prof_c4_bfs_cluster python bench.py --config c4_road --steps 1 --warmup 1 --no-cpu-baseline --no-extras \
     > $OUT/ncu_c4_bfs.log 2>&1; echo "ncu c4 bfs rc=$?"
  python scripts/ncu_summary.py $OUT/prof_c4_bfs_cluster.ncu-rep $OUT/ncu_c4_bfs_cluster_kernel.txt
  ;;
configs)
  timeout 1500 python -m pytest tests -m "gpu and slow" -x -q > $OUT/configs_tests.log 2>&1; echo "configs rc=$?"; tail -5 $OUT/configs_tests.log
  ;;
launches)
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c2_auto.csv \
     python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-extras > $OUT/launches_bench.json 2>&1; echo "launches rc=$?"
  ;;
ncu)
  for d in auto push; do
    timeout 1200 ncu --set full --clock-control none --import-source on -k regex:bfs_kernel -s 3 -c 1 \
       -o $OUT/prof_c2_$d python bench.py --steps 2 --warmup 3 --direction $d --no-cpu-baseline --no-extras \
       > $OUT/ncu_c2_$d.log 2>&1; echo "ncu c2 $d rc=$?"
    python scripts/ncu_summary.py $OUT/prof_c2_$d.ncu-rep $OUT/ncu_c2_${d}_bfs_kernel.txt
  done
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sssp_kernel -s 1 -c 1 \
     -o $OUT/prof_c3_sssp python bench.py --config c3_orkut --prim sssp --steps 1 --warmup 3 --no-cpu-baseline \
     --no-extras > $OUT/ncu_c3_sssp.log 2>&1; echo "ncu c3 sssp rc=$?"
  python scripts/ncu_summary.py $OUT/prof_c3_sssp.ncu-rep $OUT/ncu_c3_sssp_kernel.txt
  ;;
ncu_more)
  # one full capture of each session-3 kernel (one launch each; summaries next to them)
  cap() {  # name, kernel regex, skip, bench args...
    local name=$1 k=$2 sk=$3; shift 3
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $sk -c 1 \
       -o $OUT/prof_$name python bench.py --steps 1 --warmup 1 --no-cpu-baseline "$@" > $OUT/ncu_$name.log 2>&1
    echo "ncu $name rc=$?"
    python scripts/ncu_summary.py $OUT/prof_$name.ncu-rep $OUT/ncu_${name}.txt
  }
  cap c2_bc_fwd bc_fwd_kernel 2 --prim bc
  cap c2_bc_bwd bc_bwd_kernel 3 --prim bc
  cap c2_cc_hook cc_hook_csr_kernel 2 --prim cc
  cap c2_pr_adv pr_advance_kernel 4 --prim pr
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c2_bc.csv \
     python bench.py --prim bc --steps 2 --warmup 1 --no-cpu-baseline > $OUT/launches_bc_bench.json 2>&1; echo "launches bc rc=$?"
  ;;
esac
done
for f in $OUT/bench_*.json; do echo "== $f"; python -c "
import json,sys
d=json.load(open('$f')); r=d['roofline']
print(d['config']['workload'], 'value %.2f %s' % (d['value'], d['unit']), 'ms %.4f' % d['ms_per_step'],
      'frac %.4f' % r['frac'], 'e2e %.2f' % d['e2e']['value'], 'cpu', d.get('cpu_baseline', {}).get('value'))" 2>&1 | tail -1; done
