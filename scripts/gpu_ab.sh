#!/bin/bash
# A/B of the matrix formats + parity tests (run under gpurun).
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/gputests.log 2>&1; echo "tests rc=$?"
for fmt in csr sell; do
  AMGB_FORMAT=$fmt python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench_$fmt.json 2> $OUT/bench_$fmt.err
  echo "bench $fmt rc=$?"
done
BCMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$BCMD > $OUT/bench_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $OUT/launches_csr.csv $BCMD > $OUT/ncu_launches.log 2>&1
echo "ncu rc=$?"
