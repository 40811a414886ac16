#!/bin/bash
# sell_rows with the 2-byte-index value table in shared memory (A1 at 256^3): tests + A/B
OUT=gpurun_out/${TAG:-r2smtab}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_formats.py tests/test_gpu_fullsize.py tests/test_gpu_batched.py tests/test_gpu_dist.py -q -m gpu -x > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -1 $OUT/tests.log
timeout 900 python scripts/ab_inproc.py --n 256 --rounds 4 --solves 3 --variants "smtab:|;l1tab:AMGB_SELL_SMEM_TAB=0|" > $OUT/ab_256.txt 2>&1; echo "ab rc=$?"; tail -2 $OUT/ab_256.txt
for m in 1 0; do AMGB_SELL_SMEM_TAB=$m timeout 300 python scripts/class_times.py --n 256 > $OUT/classes_$m.txt 2>&1; echo "== classes AMGB_SELL_SMEM_TAB=$m"; tail -8 $OUT/classes_$m.txt | head -3; done
timeout 900 python scripts/ab_inproc.py --problem poisson_perm --n 150 --rounds 3 --solves 3 --variants "smtab:|;l1tab:AMGB_SELL_SMEM_TAB=0|" > $OUT/ab_c2.txt 2>&1; echo "abc2 rc=$?"; tail -2 $OUT/ab_c2.txt
timeout 900 python scripts/ab_inproc.py --problem convdiff --n 200 --rounds 3 --solves 3 --variants "smtab:||solver=bicgstab,relax=damped_jacobi;l1tab:AMGB_SELL_SMEM_TAB=0||solver=bicgstab,relax=damped_jacobi" > $OUT/ab_c4.txt 2>&1; echo "abc4 rc=$?"; tail -2 $OUT/ab_c4.txt
timeout 600 python bench.py --batch 4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/batch4.json 2>&1; echo "batch4 rc=$?"; tail -c 300 $OUT/batch4.json
