#!/bin/bash
# ncu --set full of the level-0 batched kernels (k = 4), CSV export only.
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || exit 1
export AMGB_NO_DEVICE_LOOP=1
PCMD="python scripts/profile_solve.py --solves 2 --batch 4"
$PCMD > $OUT/profile_b4.log 2>&1 && \
ncu --set full --clock-control none --kernel-name-base demangled \
    -k "regex:sell_tma<\(int\)1, \(bool\)1, amgb::Op(RelaxB|CgDirB|Res0B|SpmvB)" -s 20 -c 4 -o $OUT/prof_b4 $PCMD > $OUT/ncu_b4.log 2>&1
echo "ncu rc=$?"
ncu -i $OUT/prof_b4.ncu-rep --page raw --csv > $OUT/prof_b4_raw.csv 2>/dev/null
ncu -i $OUT/prof_b4.ncu-rep --page details --csv > $OUT/prof_b4_details.csv 2>/dev/null
rm -f $OUT/prof_b4.ncu-rep
tail -3 $OUT/profile_b4.log
