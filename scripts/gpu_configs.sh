#!/bin/bash
# BASELINE.json configs measured with bench.py (1 GPU) + an ncu --set full capture
# of the level-0 A-pass kernels of the headline solve (for roofline.traffic).
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || exit 1
python bench.py --problem poisson --n 32 --steps 20 --warmup 3 > $OUT/cfg_c1_poisson32.json 2> $OUT/cfg_c1.err; echo "c1 rc=$?"
python bench.py --problem poisson_perm --n 150 --steps 10 --warmup 3 > $OUT/cfg_c2_perm150.json 2> $OUT/cfg_c2.err; echo "c2 rc=$?"
python bench.py --problem poisson --n 150 --steps 10 --warmup 3 > $OUT/cfg_c2ctl_poisson150.json 2> $OUT/cfg_c2ctl.err; echo "c2ctl rc=$?"
python bench.py --problem varcoef --n 256 --steps 5 --warmup 2 > $OUT/cfg_c3_varcoef256.json 2> $OUT/cfg_c3.err; echo "c3 rc=$?"
python bench.py --problem convdiff --n 200 --steps 5 --warmup 2 > $OUT/cfg_c4_convdiff200.json 2> $OUT/cfg_c4.err; echo "c4 rc=$?"
PCMD="python scripts/profile_solve.py --solves 2"
$PCMD > $OUT/profile_plain.log 2>&1 && \
AMGB_NO_DEVICE_LOOP=1 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:OpCgDir|OpRelax<\(int\)1|sell_tma<\(int\)1, \(bool\)1, amgb::OpRes0>" -s 20 -c 3 -o $OUT/prof_a0 $PCMD > $OUT/ncu_full.log 2>&1
echo "ncu full rc=$?"
