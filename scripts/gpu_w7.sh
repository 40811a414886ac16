#!/bin/bash
OUT=gpurun_out/${TAG:-w7}; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_formats.py tests/test_gpu_fullsize.py tests/test_gpu_dict.py tests/test_gpu_parity.py -q -m gpu -x > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -1 $OUT/tests.log
timeout 1200 python scripts/ab_inproc.py --n 256 --rounds 4 --solves 3 --variants "base:|;novidx:AMGB_VIDX=0|;nodict:AMGB_NO_DICT=1|" > $OUT/ab_256.txt 2>&1; echo "ab rc=$?"; tail -3 $OUT/ab_256.txt
AMGB_VIDX=0 timeout 300 python scripts/class_times.py --n 256 > $OUT/classes_novidx.txt 2>&1; tail -7 $OUT/classes_novidx.txt
timeout 300 python scripts/class_times.py --n 256 > $OUT/classes.txt 2>&1; tail -7 $OUT/classes.txt
