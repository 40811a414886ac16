#!/bin/bash
OUT=gpurun_out/r2vix; mkdir -p $OUT
cp paper_1811_05704_b200/_lib/ab_new.so paper_1811_05704_b200/_lib/libamgb.so
timeout 1500 python -m pytest tests/test_gpu_formats.py tests/test_gpu_dist.py tests/test_gpu_batched.py tests/test_gpu_sigma.py -q -m gpu -x > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -1 $OUT/tests.log
TAG=r2vix ROUNDS=4 bash scripts/gpu_ab_lib.sh
# ncu of the level-0 relax pass of the new build
cp paper_1811_05704_b200/_lib/ab_new.so paper_1811_05704_b200/_lib/libamgb.so
export AMGB_NO_DEVICE_LOOP=1
PCMD="python scripts/profile_solve.py --solves 2"
$PCMD > $OUT/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:sell_tma.*OpRelax" -s 30 -c 1 -o $OUT/prof $PCMD > $OUT/ncu.log 2>&1
echo "ncu rc=$?"
if [ -f $OUT/prof.ncu-rep ]; then
  ncu -i $OUT/prof.ncu-rep --page raw --csv > $OUT/raw.csv 2>/dev/null
  ncu -i $OUT/prof.ncu-rep --page source --csv 2>/dev/null | head -c 3000000 > $OUT/source.csv
  rm -f $OUT/prof.ncu-rep
fi
