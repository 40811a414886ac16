#!/bin/bash
# TMA-CSR: format tests, then interleaved A/B of the format policy at 256^3 and class times
OUT=gpurun_out/${TAG:-tcsr}; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_formats.py tests/test_gpu_fullsize.py tests/test_gpu_batched.py tests/test_gpu_mixed.py tests/test_gpu_dist.py -q -m gpu -rf -x > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -5 $OUT/tests.log
timeout 900 python scripts/ab_inproc.py --n 256 --rounds 4 --solves 3 --variants "sell:AMGB_TMACSR=0|;tcsrP:AMGB_TMACSR=1|;tcsrAll:AMGB_TMACSR=2|" > $OUT/ab.txt 2>&1; echo "ab rc=$?"; tail -8 $OUT/ab.txt
for m in 0 1 2; do AMGB_TMACSR=$m timeout 300 python scripts/class_times.py --n 256 > $OUT/classes_$m.txt 2>&1; echo "== classes AMGB_TMACSR=$m"; tail -9 $OUT/classes_$m.txt; done
