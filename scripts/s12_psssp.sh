# partitioned SSSP: GPU tests, bench line, launch list (session 4)
O=gpurun_out/s14; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_dist_sssp.py -x -q > $O/dist_sssp_tests.log 2>&1; echo tests rc=$?
timeout 600 python bench.py --partitioned --config c3_orkut --prim sssp --steps 4 --warmup 3 > $O/bench_part_sssp_c3.json 2> $O/bench_part_sssp_c3.err; echo psssp rc=$?
timeout 500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_part_sssp_c3.csv python bench.py --partitioned --config c3_orkut --prim sssp --steps 1 --warmup 1 > $O/l.json 2>&1; echo l rc=$?
