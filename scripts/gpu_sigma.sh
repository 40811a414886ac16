#!/bin/bash
# SELL-C-sigma check on one B200: its bitwise tests, then A/B of the headline
# and C2 with / without sorting (AMGB_NO_SIGMA=1), then the whole GPU suite.
OUT=gpurun_out; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_sigma.py -q -x > $OUT/sg_tests.log 2>&1; echo "sigma tests rc=$?"; tail -3 $OUT/sg_tests.log
for v in 1 0 1 0; do
  if [ $v = 1 ]; then E="AMGB_SIGMA=1"; else E="AMGB_SIGMA_OFF=1"; fi
  env $E python bench.py --no-cpu-baseline --no-e2e --steps 8 > $OUT/sg_b256_$v.json 2> $OUT/sg_b256_$v.err
  python -c "import json; d=json.load(open('$OUT/sg_b256_$v.json')); print('256 sigma=$v', round(d['config']['solve_ms'],3), d['config']['iters_per_solve'], round(d['config']['solve_roofline_frac'],3), round(d['roofline']['frac'],3))"
done
for v in 1 0; do
  if [ $v = 1 ]; then E="AMGB_SIGMA=1"; else E="AMGB_SIGMA_OFF=1"; fi
  env $E python bench.py --problem poisson_perm --n 150 --no-cpu-baseline --no-e2e --steps 10 > $OUT/sg_c2_$v.json 2> $OUT/sg_c2_$v.err
  python -c "import json; d=json.load(open('$OUT/sg_c2_$v.json')); print('c2 sigma=$v', round(d['config']['solve_ms'],3), d['config']['iters_per_solve'])"
done
python scripts/class_times.py > $OUT/sg_class_times.txt 2>&1; cat $OUT/sg_class_times.txt
timeout 1200 python -m pytest tests -q -m gpu > $OUT/sg_gputests.log 2>&1; echo "gpu tests rc=$?"; tail -3 $OUT/sg_gputests.log
