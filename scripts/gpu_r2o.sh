#!/bin/bash
OUT=gpurun_out/r2o; mkdir -p $OUT
timeout 1800 python -m pytest tests -q -m gpu -rf > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -2 $OUT/tests.log; grep FAILED $OUT/tests.log | head
TAG=r2o bash scripts/gpu_configs_r2.sh
AMGB_SETUP_TIMING=1 python - > $OUT/setup.log 2>&1 <<'PY'
import time, torch, synth, paper_1811_05704_b200 as amgb
p, c, v, f = synth.problem("poisson", 256)
torch.empty(1, device="cuda"); torch.cuda.synchronize()
for k in range(2):
    t = time.perf_counter(); h = amgb.setup(p, c, v); print("setup_s", round(time.perf_counter() - t, 3), flush=True); del h
PY
grep -E "setup_s|hierarchy|device store" $OUT/setup.log
