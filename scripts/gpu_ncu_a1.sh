#!/bin/bash
# level-1 A passes (sell_rows, 2-byte value indices) at 256^3: tests of the current build,
# a short A/B against AMGB_TMACSR=4 (A1 in csr_tma), ncu --set full of the A1 res0 / relax launches
OUT=gpurun_out/${TAG:-r2a1}; mkdir -p $OUT
[ -n "$SKIP_AB" ] || timeout 900 python -m pytest tests/test_gpu_formats.py -q -m gpu -x > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -1 $OUT/tests.log
[ -n "$SKIP_AB" ] || timeout 600 python scripts/ab_inproc.py --n 256 --rounds 3 --solves 3 --variants "default:|;tmacsr4:AMGB_TMACSR=4|" > $OUT/ab_256.txt 2>&1; echo "ab rc=$?"; tail -2 $OUT/ab_256.txt
export AMGB_NO_DEVICE_LOOP=1
PCMD="python scripts/profile_solve.py --solves 1"
$PCMD > $OUT/profile_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:sell_rows<\(int\)8, \(bool\)1, \(bool\)1, amgb::OpRes0MF|sell_rows<\(int\)8, \(bool\)1, \(bool\)1, amgb::OpRelax<\(int\)0" \
    -s 4 -c 4 -o $OUT/prof_a1 $PCMD > $OUT/ncu_full.log 2>&1
echo "ncu full rc=$?"; tail -3 $OUT/ncu_full.log
if [ -f $OUT/prof_a1.ncu-rep ]; then
  ncu -i $OUT/prof_a1.ncu-rep --page raw --csv > $OUT/prof_a1_raw.csv 2>/dev/null
  ncu -i $OUT/prof_a1.ncu-rep --page details --csv > $OUT/prof_a1_details.csv 2>/dev/null
  ncu -i $OUT/prof_a1.ncu-rep --page source --csv --print-source sass > $OUT/prof_a1_source.csv 2>/dev/null
  head -c 3000000 $OUT/prof_a1_source.csv > $OUT/prof_a1_source_head.csv; rm -f $OUT/prof_a1_source.csv $OUT/prof_a1.ncu-rep
fi
