mkdir -p gpurun_out/s7
timeout 600 python -m pytest tests/test_gpu_dist.py tests/test_gpu_dist_sssp.py -x -q > gpurun_out/s7/dist_tests.log 2>&1; echo dist rc=$?
timeout 600 python bench.py --partitioned --config c5_kron25 --steps 4 --warmup 3 > gpurun_out/s7/bench_part_c5.json 2> gpurun_out/s7/bench_part_c5.err; echo part rc=$?
timeout 600 python bench.py --partitioned --keep-order --config c5_kron25 --steps 4 --warmup 3 > gpurun_out/s7/bench_part_c5_keep.json 2> gpurun_out/s7/bench_part_c5_keep.err; echo keep rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s7/launches_part_c5.csv python bench.py --partitioned --config c5_kron25 --steps 2 --warmup 1 > gpurun_out/s7/launches_part.json 2>&1; echo launches rc=$?
