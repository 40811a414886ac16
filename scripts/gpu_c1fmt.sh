#!/bin/bash
OUT=gpurun_out/${TAG:-c1fmt}; mkdir -p $OUT
timeout 900 python scripts/ab_inproc.py --n 32 --rounds 4 --solves 10 --variants "base:|;sell:AMGB_FORMAT=sell|;tma:AMGB_FORMAT=tma|;nopdl:AMGB_PDL=0|" > $OUT/ab_32.txt 2>&1; echo "ab32 rc=$?"; tail -4 $OUT/ab_32.txt
timeout 900 python scripts/ab_inproc.py --n 64 --rounds 4 --solves 5 --variants "base:|;sell:AMGB_FORMAT=sell|;pdl:AMGB_PDL=1|" > $OUT/ab_64.txt 2>&1; echo "ab64 rc=$?"; tail -3 $OUT/ab_64.txt
