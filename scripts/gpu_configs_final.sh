#!/bin/bash
# BASELINE.json configs with the round-end build (1 GPU, bench.py defaults per config).
OUT=gpurun_out/cfgf; mkdir -p $OUT
python bench.py --problem poisson --n 32 --steps 20 --warmup 3 --no-cpu-baseline > $OUT/c1_poisson32.json 2> $OUT/c1.err; echo "c1 rc=$?"
python bench.py --problem poisson_perm --n 150 --steps 10 --warmup 3 > $OUT/c2_perm150.json 2> $OUT/c2.err; echo "c2 rc=$?"
python bench.py --problem varcoef --n 256 --steps 5 --warmup 3 --no-cpu-baseline > $OUT/c3_varcoef256.json 2> $OUT/c3.err; echo "c3 rc=$?"
python bench.py --problem convdiff --n 200 --steps 5 --warmup 3 --no-cpu-baseline > $OUT/c4_convdiff200.json 2> $OUT/c4.err; echo "c4 rc=$?"
python bench.py --batch 4 --steps 5 --warmup 3 --no-cpu-baseline > $OUT/h0_batch4.json 2> $OUT/b4.err; echo "b4 rc=$?"
python bench.py --precision mixed --steps 5 --warmup 3 --no-cpu-baseline > $OUT/h0_mixed.json 2> $OUT/mx.err; echo "mixed rc=$?"
for f in $OUT/*.json; do python -c "
import json,sys; d=json.load(open('$f')); c=d['config']
print('$f'.split('/')[-1], round(d['value'],1), d['unit'], 'solve_ms', round(c.get('solve_ms',0) or 0,3), 'iters', c.get('iters_per_solve'), 'frac', round(d['roofline']['frac'],3) if d.get('roofline') else None, 'e2e', round(d['e2e']['value'],1) if d.get('e2e') else None, 'cpu', d['cpu_baseline']['value'] if d.get('cpu_baseline') else None, 'reord', c.get('reordered_store'))"; done
