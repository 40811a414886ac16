#!/bin/bash
# A/B of the shared-memory value table (size rule) on C2 / H0 / C4, then the round-end evidence
OUT=gpurun_out/r2smtab2; mkdir -p $OUT
timeout 900 python scripts/ab_inproc.py --problem poisson_perm --n 150 --rounds 3 --solves 3 --variants "rule:|;l1tab:AMGB_SELL_SMEM_TAB=0|;always:AMGB_SELL_SMEM_TAB=1|" > $OUT/ab_c2.txt 2>&1; echo "abc2 rc=$?"; tail -3 $OUT/ab_c2.txt
timeout 900 python scripts/ab_inproc.py --n 256 --rounds 4 --solves 3 --variants "rule:|;l1tab:AMGB_SELL_SMEM_TAB=0|" > $OUT/ab_256.txt 2>&1; echo "ab rc=$?"; tail -2 $OUT/ab_256.txt
timeout 900 python scripts/ab_inproc.py --problem convdiff --n 200 --rounds 3 --solves 3 --variants "rule:||solver=bicgstab,relax=damped_jacobi;l1tab:AMGB_SELL_SMEM_TAB=0||solver=bicgstab,relax=damped_jacobi" > $OUT/ab_c4.txt 2>&1; echo "abc4 rc=$?"; tail -2 $OUT/ab_c4.txt
TAG=r2_end4 TAG2=r2_final6 bash scripts/gpu_round_end.sh
