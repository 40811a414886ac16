#!/bin/bash
# GPU aggregation: setup tests (bitwise vs host builder incl. 256^3) + setup timing
OUT=gpurun_out/${TAG:-agg}; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_setup.py tests/test_gpu_dist.py tests/test_gpu_parity.py -q -m gpu -rf --durations=8 > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -12 $OUT/tests.log
for mode in gpu host; do
AMGB_SETUP_TIMING=1 python - $mode > $OUT/setup_$mode.log 2>&1 <<'PY'
import os, sys, time
if sys.argv[1] == "host": os.environ["AMGB_HOST_AGGREGATE"] = "1"
import torch, numpy as np
import paper_1811_05704_b200 as amgb, synth
p, c, v, f = synth.problem("poisson", 256)
torch.empty(1, device="cuda"); torch.cuda.synchronize()
for k in range(2):
    t = time.perf_counter(); h = amgb.setup(p, c, v); print("setup_s", round(time.perf_counter() - t, 3), flush=True); del h
PY
echo "== $mode"; grep -E "aggregat|setup_s|rounds" $OUT/setup_$mode.log | head -20
done
