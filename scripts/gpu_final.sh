#!/bin/bash
# Round-end evidence on one B200: GPU tests, full bench (CPU baseline, e2e), the
# reference arm, the ncu launch list of the bench command, ncu --set full of the
# level-0 A passes (CSV exports), configs.
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/final_build.log 2>&1 || exit 1
timeout 1500 python -m pytest tests -q -m gpu > $OUT/final_gputests.log 2>&1; echo "tests rc=$?"; tail -2 $OUT/final_gputests.log
python bench.py > $OUT/final_bench.json 2> $OUT/final_bench.err; echo "bench rc=$?"
python bench.py --impl reference --steps 3 --warmup 3 > $OUT/final_reference.json 2> $OUT/final_reference.err; echo "ref rc=$?"
export AMGB_NO_DEVICE_LOOP=1
BCMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$BCMD > $OUT/final_bench_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $OUT/final_launches.csv $BCMD > $OUT/final_ncu_launches.log 2>&1
echo "ncu launches rc=$?"
PCMD="python scripts/profile_solve.py --solves 2"
$PCMD > $OUT/final_profile_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:OpCgDir|OpRelax<\(int\)1|sell_tma<\(int\)1, \(bool\)1, amgb::OpRes0|sell_tma<\(int\)1, \(bool\)1, amgb::OpProl0|VCgUpdate" \
    -s 25 -c 6 -o $OUT/final_a0 $PCMD > $OUT/final_ncu_full.log 2>&1
echo "ncu full rc=$?"
ncu -i $OUT/final_a0.ncu-rep --page raw --csv > $OUT/final_a0_raw.csv 2>/dev/null
ncu -i $OUT/final_a0.ncu-rep --page details --csv > $OUT/final_a0_details.csv 2>/dev/null
rm -f $OUT/final_a0.ncu-rep
