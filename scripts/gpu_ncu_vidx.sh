#!/bin/bash
# ncu --set full of the level-0 relax+rho pass (sell_tma) with and without value indexing
OUT=gpurun_out/${TAG:-ncuv}; mkdir -p $OUT
export AMGB_NO_DEVICE_LOOP=1
PCMD="python scripts/profile_solve.py --solves 2"
for v in vidx novidx; do
  if [ $v = vidx ]; then unset AMGB_VIDX; else export AMGB_VIDX=0; fi
  $PCMD > $OUT/plain_$v.log 2>&1 && \
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:sell_tma.*OpRelax" -s 30 -c 2 -o $OUT/prof_$v $PCMD > $OUT/ncu_$v.log 2>&1
  echo "ncu $v rc=$?"
  if [ -f $OUT/prof_$v.ncu-rep ]; then
    ncu -i $OUT/prof_$v.ncu-rep --page raw --csv > $OUT/raw_$v.csv 2>/dev/null
    ncu -i $OUT/prof_$v.ncu-rep --page details --csv > $OUT/details_$v.csv 2>/dev/null
    ncu -i $OUT/prof_$v.ncu-rep --page source --csv 2>/dev/null | head -c 4000000 > $OUT/source_$v.csv
    rm -f $OUT/prof_$v.ncu-rep
  fi
done
