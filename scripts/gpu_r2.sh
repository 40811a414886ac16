#!/bin/bash
# Round-2 GPU check: full GPU test suite (failures listed, durations), smoke(),
# and the headline bench line.  Outputs under gpurun_out/$TAG/.
TAG=${TAG:-r2}
OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt 2>&1
timeout 2400 python -m pytest tests -q -m gpu -rf --durations=15 ${PYTEST_ARGS} > $OUT/gputests.log 2>&1; echo "tests rc=$?"
tail -25 $OUT/gputests.log | grep -E "passed|failed|FAILED|Error" | head -20
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 $OUT/smoke.log
if [ -z "$NO_BENCH" ]; then
timeout 900 python bench.py --steps ${STEPS:-10} --warmup 3 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
python - $OUT/bench.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
c = d['config']
print("headline", round(d['value'], 1), d['unit'], "ms/solve", round(c['solve_ms'], 3), "it", c['iters_per_solve'],
      "A0 frac", round(d['roofline']['frac'], 3), "solve frac", round(c['solve_roofline_frac'], 3), "clk", d['clocks'],
      "e2e", round((d.get('e2e') or {}).get('value', 0), 1), "parity", d.get('parity_full_size'),
      "cpu", d.get('cpu_baseline'))
PY
fi
