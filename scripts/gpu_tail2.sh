#!/bin/bash
OUT=gpurun_out/${TAG:-tail2}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_policy.py tests/test_gpu_parity.py -q -m gpu -x > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -2 $OUT/tests.log
AMGB_TAIL=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_policy.py tests/test_gpu_formats.py -q -m gpu -x > $OUT/tests_tail.log 2>&1; echo "tests (tail on) rc=$?"; tail -2 $OUT/tests_tail.log
for n in 32 150; do
timeout 900 python scripts/ab_inproc.py --n $n --rounds 4 --solves 5 --variants "notail:|;cg2:AMGB_TAIL=1,AMGB_TAIL_BARRIER=cg,AMGB_TAIL_BLOCKS=2|;own1:AMGB_TAIL=1,AMGB_TAIL_BLOCKS=1|;own2:AMGB_TAIL=1,AMGB_TAIL_BLOCKS=2|;cg1:AMGB_TAIL=1,AMGB_TAIL_BARRIER=cg,AMGB_TAIL_BLOCKS=1|" > $OUT/ab_$n.txt 2>&1; echo "ab $n rc=$?"; tail -6 $OUT/ab_$n.txt
done
