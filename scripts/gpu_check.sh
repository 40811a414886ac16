#!/bin/bash
# Build, GPU tests, headline bench and the configs listed in CFGS (bench args, ';'-separated).
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/gputests.log 2>&1; echo "tests rc=$?"; tail -2 $OUT/gputests.log
python bench.py ${HEAD_ARGS:---no-cpu-baseline} > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d = json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1])
print("headline", d['value'], d['unit'], "ms/solve", d['config']['solve_ms'], "it", d['config']['iters_per_solve'], "frac", round(d['roofline']['frac'], 3), "clk", d['clocks'], "e2e", (d.get('e2e') or {}).get('value'))
PY
IFS=';' read -ra CF <<< "${CFGS}"
i=0
for c in "${CF[@]}"; do
  i=$((i+1))
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e $c > $OUT/cfg_$i.json 2> $OUT/cfg_$i.err
  python - "$c" "$OUT/cfg_$i.json" <<'PY'
import json, sys
d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
print(f"[{sys.argv[1]}] ms {d['config']['solve_ms']:.2f} it {d['config']['iters_per_solve']} frac {d['roofline']['frac']:.3f} clk {d['clocks']['sm_mhz']}")
PY
done
