#!/bin/bash
# 2-byte value indices in the TMA-CSR kernel (wide coarse A in csr_tma): tests + A/B
OUT=gpurun_out/${TAG:-r2vi16}; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_formats.py tests/test_gpu_fullsize.py tests/test_gpu_dist.py tests/test_gpu_batched.py tests/test_gpu_mixed.py tests/test_gpu_sigma.py tests/test_gpu_reorder.py -q -m gpu -x > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -1 $OUT/tests.log
timeout 900 python scripts/ab_inproc.py --n 256 --rounds 4 --solves 3 --variants "vi16:|;un4:AMGB_TCSR_UN=4|;old3:AMGB_TMACSR=3,AMGB_TCSR_UN=4|;old3un8:AMGB_TMACSR=3|" > $OUT/ab_256.txt 2>&1; echo "ab rc=$?"; tail -4 $OUT/ab_256.txt
for m in 3 4; do AMGB_TMACSR=$m timeout 300 python scripts/class_times.py --n 256 > $OUT/classes_$m.txt 2>&1; echo "== classes AMGB_TMACSR=$m"; tail -9 $OUT/classes_$m.txt; done
timeout 900 python scripts/ab_inproc.py --problem convdiff --n 200 --rounds 3 --solves 3 --variants "vi16:||solver=bicgstab,relax=damped_jacobi;old3:AMGB_TMACSR=3,AMGB_TCSR_UN=4||solver=bicgstab,relax=damped_jacobi" > $OUT/ab_c4.txt 2>&1; echo "abc4 rc=$?"; tail -2 $OUT/ab_c4.txt
timeout 900 python scripts/ab_inproc.py --problem poisson_perm --n 150 --rounds 3 --solves 3 --variants "vi16:|;old3:AMGB_TMACSR=3,AMGB_TCSR_UN=4|" > $OUT/ab_c2.txt 2>&1; echo "abc2 rc=$?"; tail -2 $OUT/ab_c2.txt
timeout 900 python scripts/ab_inproc.py --problem varcoef --n 256 --rounds 2 --solves 2 --variants "vi16:||relax=chebyshev;old3:AMGB_TMACSR=3,AMGB_TCSR_UN=4||relax=chebyshev" > $OUT/ab_c3.txt 2>&1; echo "abc3 rc=$?"; tail -2 $OUT/ab_c3.txt
