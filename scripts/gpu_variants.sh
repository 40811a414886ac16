#!/bin/bash
# Build, parity tests, bench variants (env settings), launch list of the default.
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/gputests.log 2>&1; echo "tests rc=$?"; tail -2 $OUT/gputests.log
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
i=0
for v in $VARIANTS; do
  i=$((i+1))
  env $v python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench_v$i.json 2> $OUT/bench_v$i.err; echo "variant $v rc=$?"
done
BCMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$BCMD > $OUT/bench_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $OUT/launches.csv $BCMD > $OUT/ncu_launches.log 2>&1
echo "ncu launches rc=$?"
