#!/bin/bash
OUT=gpurun_out/r2tc2; mkdir -p $OUT
timeout 900 python scripts/ab_inproc.py --n 256 --rounds 4 --solves 3 --variants "base:|;tcsr2:AMGB_TMACSR=2|" > $OUT/ab_256.txt 2>&1; echo "ab rc=$?"; tail -2 $OUT/ab_256.txt
AMGB_TMACSR=2 timeout 300 python scripts/class_times.py --n 256 > $OUT/classes_tcsr2.txt 2>&1; tail -7 $OUT/classes_tcsr2.txt
timeout 300 python scripts/class_times.py --n 256 > $OUT/classes.txt 2>&1; tail -7 $OUT/classes.txt
