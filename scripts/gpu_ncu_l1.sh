#!/bin/bash
# ncu --set full of the level-1 (SELL-32) kernels of the 256^3 solve; only the
# raw-page CSV comes back (the report itself is too large for gpurun_out).
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || exit 1
export AMGB_NO_DEVICE_LOOP=1
PCMD="python scripts/profile_solve.py --solves 2"
$PCMD > $OUT/profile_plain.log 2>&1 && \
ncu --set full --clock-control none --kernel-name-base demangled \
    -k "regex:${NCU_REGEX:-sell_rows}" -s ${NCU_SKIP:-24} -c ${NCU_COUNT:-6} -o /tmp/prof_l1 $PCMD > $OUT/ncu_l1.log 2>&1
echo "ncu rc=$?"
ncu -i /tmp/prof_l1.ncu-rep --page raw --csv > $OUT/prof_l1_raw.csv 2>/dev/null
ncu -i /tmp/prof_l1.ncu-rep --page details --csv > $OUT/prof_l1_details.csv 2>/dev/null
ls -la $OUT
