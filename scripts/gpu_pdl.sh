#!/bin/bash
OUT=gpurun_out/${TAG:-pdl}; mkdir -p $OUT
for n in 32 150 256; do
timeout 900 python scripts/ab_inproc.py --n $n --rounds 4 --solves 5 --variants "base:|;pdl:AMGB_PDL=1|" > $OUT/ab_$n.txt 2>&1; echo "ab $n rc=$?"; tail -2 $OUT/ab_$n.txt
done
