#!/bin/bash
# A/B an env toggle (AB_VAR) on the headline bench after the GPU parity tests.
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/gputests.log 2>&1; echo "tests rc=$?"; tail -2 $OUT/gputests.log
for rep in 1 2; do
  for v in 0 1; do
    if [ $v = 1 ]; then export $AB_VAR=1; else unset $AB_VAR; fi
    python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS} > $OUT/bench_ab_${v}_${rep}.json 2> $OUT/bench_ab_${v}_${rep}.err
    python - "$v" "$OUT/bench_ab_${v}_${rep}.json" <<'PY'
import json, sys
d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
print(f"off_or_on={sys.argv[1]} ms/solve {d['config'].get('solve_ms')} iters {d['config'].get('iters_per_solve')} value {d['value']:.1f} frac {d['roofline']['frac']:.3f} mhz {d['clocks']['sm_mhz']}")
PY
  done
done
unset $AB_VAR
