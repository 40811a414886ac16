#!/bin/bash
# Measurement sweep of the §8 rows on one B200 (JSON lines into gpurun_out/sweep_*.json).
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || exit 1
run() {  # name, args
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e $2 > $OUT/sweep_$1.json 2> $OUT/sweep_$1.err
  python - "$1" "$OUT/sweep_$1.json" <<'PY'
import json, sys
d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
c = d['config']
print(f"{sys.argv[1]:14s} {d['value']:9.1f} {d['unit']:14s} ms {c.get('solve_ms'):8.2f} it {c.get('iters_per_solve')} "
      f"alg {c.get('solve_alg_GBps', 0)/1e3:.2f} TB/s frac {d['roofline'].get('frac')} clk {d['clocks']['sm_mhz']}")
PY
}
run c1_poisson32 "--problem poisson --n 32"
run batch2 "--batch 2"
run batch4 "--batch 4"
run batch8 "--batch 8"
run mixed "--precision mixed"
run mixed_perm150 "--precision mixed --problem poisson_perm --n 150"
run jacobi256 "--relax damped_jacobi"
run idrs_poisson256 "--solver idrs"
