#!/bin/bash
# Env-toggle bisection of a bench config (BENCH_ARGS) without rebuilding.
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || exit 1
for v in "" "AMGB_NO_CG_FUSION=1" "AMGB_NO_MF=1" "AMGB_NO_DICT=1" "AMGB_NO_CG_FUSION=1 AMGB_NO_MF=1" ; do
  for args in "--problem poisson_perm --n 150" "--problem poisson --n 150"; do
    env $v python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e $args > $OUT/bis.json 2> $OUT/bis.err
    python - "$v" "$args" <<'PY'
import json, sys
d = json.loads(open('gpurun_out/bis.json').read().strip().splitlines()[-1])
print(f"[{sys.argv[1]}] [{sys.argv[2]}] ms {d['config']['solve_ms']:.2f} it {d['config']['iters_per_solve']} mhz {d['clocks']['sm_mhz']}")
PY
  done
done
