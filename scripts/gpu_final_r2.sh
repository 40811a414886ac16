#!/bin/bash
# Round-2 final evidence on one B200: GPU tests, smoke, the driver's bench lines
# (product and reference arm), the ncu launch list of the bench command and one
# ncu --set full capture of the level-0 A passes (roofline.traffic, with the
# profiled library's sha256).  Outputs under gpurun_out/$TAG.
TAG=${TAG:-final}
OUT=gpurun_out/$TAG; mkdir -p $OUT
sha256sum paper_1811_05704_b200/_lib/libamgb.so | cut -d' ' -f1 > $OUT/lib_sha256.txt
if [ -z "$SKIP_TESTS" ]; then
timeout 2400 python -m pytest tests -q -m gpu -rf --durations=15 > $OUT/gputests.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/gputests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $OUT/smoke.log
fi
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
python - $OUT/bench.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
c = d['config']; r = d['roofline']
print("headline", round(d['value'], 1), d['unit'], "ms/solve", round(c['solve_ms'], 3), "it", c['iters_per_solve'],
      "A0 frac", round(r['frac'], 3), "GB/launch", round(r['bytes_per_launch'] / 1e9, 3), "ms/launch", round(r['ms_per_launch'], 4),
      "solve frac", round(c['solve_roofline_frac'], 3), "clk", d['clocks'], "e2e", round(d['e2e']['value'], 1),
      "parity", d['parity_full_size'], "cpu", d['cpu_baseline']['value'], "setup_s", round(c['setup_s'], 2))
PY
if [ -z "$SKIP_REF" ]; then
timeout 1200 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $OUT/ref.json 2> $OUT/ref.err; echo "ref rc=$?"; tail -c 400 $OUT/ref.json
fi
# the other BASELINE configs with clock records
[ -n "$SKIP_CFG" ] || TAG=$TAG bash scripts/gpu_configs_r2.sh
# ncu: launch list of the bench command (host loop over the iteration graph: ncu does not
# enumerate kernels inside conditional graph nodes), then --set full on the level-0 A passes
export AMGB_NO_DEVICE_LOOP=1
BCMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$BCMD > $OUT/bench_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $OUT/launches.csv $BCMD > $OUT/ncu_launches.log 2>&1
echo "ncu launches rc=$?"
python scripts/summarize_launches.py $OUT/launches.csv > $OUT/launches_summary.txt 2>&1; head -40 $OUT/launches_summary.txt
PCMD="python scripts/profile_solve.py --solves 2"
$PCMD > $OUT/profile_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:sell_tma.*(OpCgDir|OpRelax<\(int\)1|OpRes0)|csr_tma.*OpProl0|sell_rows.*OpSpmvMF|VCgUpdate" \
    -s 25 -c 6 -o $OUT/prof_a0 $PCMD > $OUT/ncu_full.log 2>&1
echo "ncu full rc=$?"
if [ -f $OUT/prof_a0.ncu-rep ]; then
  ncu -i $OUT/prof_a0.ncu-rep --page raw --csv > $OUT/prof_a0_raw.csv 2>/dev/null
  ncu -i $OUT/prof_a0.ncu-rep --page details --csv > $OUT/prof_a0_details.csv 2>/dev/null
  rm -f $OUT/prof_a0.ncu-rep
fi
