#!/bin/bash
OUT=gpurun_out/r02f; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_pbfs.py -x -q > $OUT/pbfs_tests.log 2>&1; echo "pbfs tests rc=$?"; tail -30 $OUT/pbfs_tests.log
