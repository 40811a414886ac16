#!/bin/bash
# BASELINE configs on one B200 with clock records: C1 32^3, C2 150^3 permuted, C3 256^3 var-coef
# Chebyshev, C4 200^3 conv-diff BiCGStab, H0 batched k = 4, H0 mixed precision
OUT=gpurun_out/${TAG:-cfg}; mkdir -p $OUT
run() {  # name args...
  local name=$1; shift
  timeout 900 python bench.py --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-e2e "$@" > $OUT/$name.json 2> $OUT/$name.err
  python - $OUT/$name.json $name <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); c = d['config']
r = d.get('roofline') or {}
print(f"{sys.argv[2]:10s} {c.get('solve_ms', d['ms_per_step']):9.3f} ms  {d['value']:9.1f} {d['unit']:22s} it {c.get('iters_per_solve', c.get('iters_per_column'))}  "
      f"A0frac {r.get('frac') if r.get('frac') is None else round(r['frac'], 3)}  solvefrac {round(c.get('solve_roofline_frac', 0), 3)}  clk {d['clocks']['sm_mhz']} {d['clocks']['reasons']}")
PY
}
run c1 --n 32 --steps 50
run c2 --problem poisson_perm --n 150
run c3 --problem varcoef --n 256
run c4 --problem convdiff --n 200
run h0_batch4 --batch 4
run h0_mixed --precision mixed
