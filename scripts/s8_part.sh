# partitioned BFS/SSSP: GPU dist tests, bench lines, launch list (session 4)
O=gpurun_out/s8; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_dist.py tests/test_gpu_dist_sssp.py -x -q > $O/dist_tests.log 2>&1; echo dist rc=$?
timeout 600 python bench.py --partitioned --config c5_kron25 --steps 4 --warmup 3 > $O/bench_part_c5.json 2> $O/bench_part_c5.err; echo part rc=$?
timeout 600 python bench.py --partitioned --config c3_orkut --prim sssp --steps 4 --warmup 3 > $O/bench_part_sssp_c3.json 2> $O/bench_part_sssp_c3.err; echo psssp rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_part_c5.csv python bench.py --partitioned --config c5_kron25 --steps 2 --warmup 1 > $O/launches_part.json 2>&1; echo launches rc=$?
