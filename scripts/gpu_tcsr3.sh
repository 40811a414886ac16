#!/bin/bash
OUT=gpurun_out/r2tc3; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_formats.py tests/test_gpu_fullsize.py tests/test_gpu_dist.py tests/test_gpu_batched.py tests/test_gpu_mixed.py tests/test_gpu_sigma.py tests/test_gpu_reorder.py -q -m gpu -x > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -1 $OUT/tests.log
timeout 900 python scripts/ab_inproc.py --n 256 --rounds 4 --solves 3 --variants "wideR:|;narrowonly:AMGB_TMACSR=1|" > $OUT/ab_256.txt 2>&1; echo "ab rc=$?"; tail -2 $OUT/ab_256.txt
timeout 900 python scripts/ab_inproc.py --problem convdiff --n 200 --rounds 3 --solves 3 --variants "wideR:|;narrowonly:AMGB_TMACSR=1|" > $OUT/ab_c4.txt 2>&1; echo "abc4 rc=$?"; tail -2 $OUT/ab_c4.txt
timeout 900 python scripts/ab_inproc.py --problem poisson_perm --n 150 --rounds 3 --solves 3 --variants "wideR:|;narrowonly:AMGB_TMACSR=1|" > $OUT/ab_c2.txt 2>&1; echo "abc2 rc=$?"; tail -2 $OUT/ab_c2.txt
