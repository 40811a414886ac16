#!/bin/bash
# In-graph per-class solve time at the final HEAD (256^3 Poisson; C4 conv-diff 200^3).
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/cls_build.log 2>&1 || exit 1
timeout 600 python scripts/class_times.py --problem poisson --n 256 > $OUT/cls_poisson256.txt 2>&1; echo "p256 rc=$?"
timeout 600 python scripts/class_times.py --problem poisson_perm --n 150 > $OUT/cls_perm150.txt 2>&1; echo "c2 rc=$?"
