#!/bin/bash
# A/B of two library builds on one box (_lib/ab_{old,new}.so, interleaved processes):
# the 256^3 headline bench solve time per build, ROUNDS rounds.
OUT=gpurun_out/${TAG:-ablib}; mkdir -p $OUT
LIB=paper_1811_05704_b200/_lib/libamgb.so
D=paper_1811_05704_b200/_lib
for round in $(seq 1 ${ROUNDS:-3}); do
  for v in old new; do
    cp $D/ab_$v.so $LIB
    python bench.py --no-cpu-baseline --no-e2e --steps 10 > $OUT/ab_$v$round.json 2> $OUT/ab_$v$round.err
    python -c "import json; d=json.loads(open('$OUT/ab_$v$round.json').read().splitlines()[-1]); print('$v', round(d['config']['solve_ms'],3), d['config']['iters_per_solve'], d['clocks']['sm_mhz'], round(d['roofline']['ms_per_launch'],4))"
  done
done
cp $D/ab_new.so $LIB
