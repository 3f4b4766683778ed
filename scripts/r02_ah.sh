#!/bin/bash
OUT=gpurun_out/r02ah; mkdir -p $OUT
for lib in libgr_b200.so libgr_nostay.so libgr_b200.so libgr_nostay.so; do
  GR_LIB=$lib timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-extras 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('c2 $lib', d['ms_per_step'], d['levels_per_step'])"
done
for lib in libgr_b200.so libgr_nostay.so; do
  GR_LIB=$lib timeout 600 python bench.py --config c3_orkut --steps 10 --warmup 3 --no-cpu-baseline --no-extras 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('c3 $lib', d['ms_per_step'], d['levels_per_step'])"
  GR_LIB=$lib timeout 600 python bench.py --config c5_kron25 --steps 8 --warmup 3 --no-cpu-baseline --no-extras 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('c5 $lib', d['ms_per_step'], d['levels_per_step'])"
  GR_LIB=$lib timeout 600 python bench.py --config c1_rmat16 --steps 10 --warmup 3 --no-cpu-baseline --no-extras 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('c1 $lib', d['ms_per_step'], d['levels_per_step'])"
done
