#!/bin/bash
# value-indexed storage: tests, interleaved A/B vs the fp64-array store, class times, bench line
OUT=gpurun_out/${TAG:-vidx}; mkdir -p $OUT
timeout 2000 python -m pytest tests -q -m gpu -rf --durations=10 > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -4 $OUT/tests.log | head -3; grep FAILED $OUT/tests.log | head
timeout 900 python scripts/ab_inproc.py --n 256 --rounds 4 --solves 3 --variants "vidx:|;plain:AMGB_NO_VIDX=1|" > $OUT/ab_256.txt 2>&1; echo "ab256 rc=$?"; tail -2 $OUT/ab_256.txt
timeout 900 python scripts/ab_inproc.py --problem convdiff --n 200 --rounds 3 --solves 3 --variants "vidx:|;plain:AMGB_NO_VIDX=1|" > $OUT/ab_c4.txt 2>&1; echo "abc4 rc=$?"; tail -2 $OUT/ab_c4.txt
timeout 300 python scripts/class_times.py --n 256 > $OUT/classes.txt 2>&1; tail -7 $OUT/classes.txt
timeout 900 python bench.py --steps 10 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
python - $OUT/bench.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
c = d['config']
print("headline", round(d['value'], 1), d['unit'], "ms/solve", round(c['solve_ms'], 3), "it", c['iters_per_solve'],
      "A0 frac", round(d['roofline']['frac'], 3), "A0 GB/launch", round(d['roofline']['bytes_per_launch']/1e9, 3), "solve frac", round(c['solve_roofline_frac'], 3), "clk", d['clocks'],
      "e2e", round((d.get('e2e') or {}).get('value', 0), 1), "parity", d.get('parity_full_size'))
PY
