#!/bin/bash
# ncu evidence on one B200: the launch list of the bench command and a --set full
# capture of the level-0 A-pass kernels.  AMGB_NO_DEVICE_LOOP=1 because ncu cannot
# profile kernels inside a graph that has conditional nodes (the timed path uses one).
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/gputests.log 2>&1; echo "tests rc=$?"; tail -2 $OUT/gputests.log
export AMGB_NO_DEVICE_LOOP=1
BCMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$BCMD > $OUT/bench_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $OUT/launches.csv $BCMD > $OUT/ncu_launches.log 2>&1
echo "ncu launches rc=$?"
PCMD="python scripts/profile_solve.py --solves 2"
$PCMD > $OUT/profile_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:OpCgDir|OpRelax<\(int\)1|sell_tma<\(int\)1, \(bool\)1, amgb::OpRes0>|sell_tma<\(int\)1, \(bool\)1, amgb::OpProl0>|VCgUpdate" \
    -s 25 -c 5 -o $OUT/prof_a0 $PCMD > $OUT/ncu_full.log 2>&1
echo "ncu full rc=$?"
if [ -f $OUT/prof_a0.ncu-rep ]; then
  ncu -i $OUT/prof_a0.ncu-rep --page raw --csv > $OUT/prof_a0_raw.csv 2>/dev/null
  ncu -i $OUT/prof_a0.ncu-rep --page details --csv > $OUT/prof_a0_details.csv 2>/dev/null
  [ -n "$KEEP_REP" ] || rm -f $OUT/prof_a0.ncu-rep
fi
