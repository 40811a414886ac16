#!/bin/bash
OUT=gpurun_out/r2tct; mkdir -p $OUT
cp paper_1811_05704_b200/_lib/ab_new.so paper_1811_05704_b200/_lib/libamgb.so
timeout 1500 python -m pytest tests/test_gpu_formats.py tests/test_gpu_dist.py tests/test_gpu_batched.py tests/test_gpu_mixed.py -q -m gpu -x > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -1 $OUT/tests.log
TAG=r2tct ROUNDS=4 bash scripts/gpu_ab_lib.sh
