#!/bin/bash
# A/B of the shipped build (_lib/ab_old.so) against the no-split-compile build with the
# shared-memory SELL table (_lib/ab_new.so), interleaved processes; the faster one stays,
# and the new one gets the round-end evidence if it wins
OUT=gpurun_out/r2ns; mkdir -p $OUT
D=paper_1811_05704_b200/_lib
nvidia-smi --query-gpu=name,serial,pci.bus_id --format=csv > $OUT/box.txt 2>&1
for round in 1 2; do
  for v in old new; do
    cp $D/ab_$v.so $D/libamgb.so
    timeout 300 python scripts/class_times.py --n 256 > $OUT/classes_${v}_$round.txt 2>&1
    echo "== $v round $round"; grep -E "unprofiled|transfer|A coarse|A0 pass" $OUT/classes_${v}_$round.txt
  done
done
python - $OUT <<'PY' > $OUT/winner.txt
import re, sys, glob
t = {}
for f in glob.glob(sys.argv[1] + "/classes_*_*.txt"):
    v = f.split("classes_")[1].split("_")[0]
    m = re.search(r"unprofiled solve: ([\d.]+) ms", open(f).read())
    if m: t.setdefault(v, []).append(float(m.group(1)))
old, new = sum(t["old"]) / len(t["old"]), sum(t["new"]) / len(t["new"])
print("new" if new < old - 0.15 else "old", round(old, 3), round(new, 3))
PY
cat $OUT/winner.txt
if [ "$(cut -d' ' -f1 $OUT/winner.txt)" = "new" ]; then
  cp $D/ab_new.so $D/libamgb.so
  TAG=r2_final9 bash scripts/gpu_final_r2.sh
else
  cp $D/ab_old.so $D/libamgb.so
fi
