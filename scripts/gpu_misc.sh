#!/bin/bash
# csr_tma unroll A/B, PDL A/B, setup timing at 256^3
OUT=gpurun_out/${TAG:-misc}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_formats.py -q -m gpu -x -k "per_row and (auto or tmacsr)" > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -1 $OUT/tests.log
timeout 900 python scripts/ab_inproc.py --n 256 --rounds 4 --solves 3 --variants "un4:|;un8:AMGB_TCSR_UN=8|;pdl:AMGB_PDL=1|" > $OUT/ab_256.txt 2>&1; echo "ab256 rc=$?"; tail -3 $OUT/ab_256.txt
for n in 32 150; do
timeout 900 python scripts/ab_inproc.py --n $n --rounds 4 --solves 5 --variants "base:|;pdl:AMGB_PDL=1|" > $OUT/ab_$n.txt 2>&1; echo "ab $n rc=$?"; tail -2 $OUT/ab_$n.txt
done
AMGB_SETUP_TIMING=1 python - > $OUT/setup.log 2>&1 <<'PY'
import time, torch, synth, paper_1811_05704_b200 as amgb
p, c, v, f = synth.problem("poisson", 256)
torch.empty(1, device="cuda"); torch.cuda.synchronize()
for k in range(2):
    t = time.perf_counter(); h = amgb.setup(p, c, v); print("setup_s", round(time.perf_counter() - t, 3), flush=True); del h
PY
grep -E "setup_s|hierarchy|device store|vidx|matrix" $OUT/setup.log | tail -20
