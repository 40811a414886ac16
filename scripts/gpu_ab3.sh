#!/bin/bash
# three library builds on one box, interleaved processes: class times at 256^3 (same env)
OUT=gpurun_out/${TAG:-r2ab3}; mkdir -p $OUT
D=paper_1811_05704_b200/_lib
export AMGB_TMACSR=3 AMGB_TCSR_UN=4
for round in 1 2; do
  for v in old vi16 cur; do
    cp $D/ab_$v.so $D/libamgb.so
    timeout 300 python scripts/class_times.py --n 256 > $OUT/classes_${v}_$round.txt 2>&1
    echo "== $v round $round"; grep -E "unprofiled|transfer|A coarse|A0 pass" $OUT/classes_${v}_$round.txt
  done
done
cp $D/ab_cur.so $D/libamgb.so
