#!/bin/bash
# A/B of two library builds (abtmp/libamgb_{old,new}.so, interleaved) on C4:
# conv-diff 200^3, BiCGStab + damped Jacobi.
OUT=gpurun_out; mkdir -p $OUT
LIB=paper_1811_05704_b200/_lib/libamgb.so
for round in 1 2 3; do
  for v in old new; do
    cp abtmp/libamgb_$v.so $LIB
    python bench.py --problem convdiff --n 200 --solver bicgstab --relax damped_jacobi --no-cpu-baseline --no-e2e --steps 8 > $OUT/c4ab_$v$round.json 2> $OUT/c4ab_$v$round.err
    python -c "import json; d=json.load(open('$OUT/c4ab_$v$round.json')); print('$v', round(d['config']['solve_ms'],3), d['config']['iters_per_solve'], d['clocks']['sm_mhz'])"
  done
done
cp abtmp/libamgb_new.so $LIB
