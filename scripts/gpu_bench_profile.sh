#!/bin/bash
# Round measurement on one B200 (run under gpurun from the repo root):
#   1. build, 2. bench.py (plain), 3. ncu launch list of the same bench command,
#   4. ncu --set full of the level-0 A-pass kernels on a short solve driver.
set -x
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || exit 1
python bench.py --steps ${STEPS:-10} --warmup ${WARMUP:-3} > $OUT/bench.json 2> $OUT/bench.err
echo "bench rc=$?"
BCMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$BCMD > $OUT/bench_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $OUT/launches.csv $BCMD > $OUT/ncu_launches.log 2>&1
echo "ncu launches rc=$?"
PCMD="python scripts/profile_solve.py --solves 2"
$PCMD > $OUT/profile_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sell_rows -s 60 -c 4 -o $OUT/prof_a0 $PCMD > $OUT/ncu_full.log 2>&1
echo "ncu full rc=$?"
