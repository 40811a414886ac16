#!/bin/bash
# Quick refresh on one B200: build + smoke, GPU tests, default bench, C2 with the
# library's default (automatic) reordering and with reordering off.
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/rf_build.log 2>&1 || { tail -20 $OUT/rf_build.log; exit 1; }
timeout 1200 python -m pytest tests -q -m gpu > $OUT/rf_gputests.log 2>&1; echo "tests rc=$?"; tail -2 $OUT/rf_gputests.log
python bench.py > $OUT/rf_bench.json 2> $OUT/rf_bench.err; echo "bench rc=$?"
python bench.py --problem poisson_perm --n 150 --steps 10 --warmup 3 --no-cpu-baseline > $OUT/rf_c2auto.json 2> $OUT/rf_c2auto.err; echo "c2 auto rc=$?"
python bench.py --problem poisson_perm --n 150 --steps 10 --warmup 3 --no-cpu-baseline --reorder off > $OUT/rf_c2off.json 2> $OUT/rf_c2off.err; echo "c2 off rc=$?"
for f in rf_bench rf_c2auto rf_c2off; do python -c "import json,sys; d=json.load(open('$OUT/$f.json')); print('$f', d['value'], d['config'].get('solve_ms'), d['config'].get('iters_per_solve'), d['roofline']['frac'], d['config'].get('reordered_store'))"; done
