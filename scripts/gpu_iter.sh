#!/bin/bash
# Iteration loop on one B200: build, GPU parity tests, bench (no CPU baseline),
# ncu launch list, and an ncu --set full capture of the level-0 A-pass kernels.
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/gputests.log 2>&1; echo "tests rc=$?"; tail -2 $OUT/gputests.log
python bench.py --steps 10 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
BCMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e ${BENCH_ARGS}"
if [ -z "$NO_LAUNCHES" ]; then
$BCMD > $OUT/bench_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $OUT/launches.csv $BCMD > $OUT/ncu_launches.log 2>&1
echo "ncu launches rc=$?"
fi
if [ -n "$NCU_FULL" ]; then
PCMD="python scripts/profile_solve.py --solves 2"
$PCMD > $OUT/profile_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:${NCU_REGEX:-OpCgDir|OpRelax<1|OpRes0}" -s ${NCU_SKIP:-30} -c ${NCU_COUNT:-6} -o $OUT/prof_full $PCMD > $OUT/ncu_full.log 2>&1
echo "ncu full rc=$?"
fi
