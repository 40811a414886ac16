#!/bin/bash
# Tail cycle: parity tests, then A/B (AMGB_NO_TAIL) on C1 32^3, 150^3 and 256^3, and a C1 bench line
OUT=gpurun_out/${TAG:-tail}; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_formats.py tests/test_gpu_policy.py tests/test_gpu_reorder.py tests/test_gpu_host_stream.py tests/test_gpu_gmres.py tests/test_gpu_idrs.py tests/test_gpu_setup.py -q -m gpu -rf -x > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -5 $OUT/tests.log
for n in 32 150 256; do
timeout 900 python scripts/ab_inproc.py --n $n --rounds 4 --solves 5 --variants "tail:|;notail:AMGB_NO_TAIL=1|" > $OUT/ab_$n.txt 2>&1; echo "ab $n rc=$?"; tail -3 $OUT/ab_$n.txt
done
timeout 600 python bench.py --n 32 --steps 50 --warmup 5 --no-cpu-baseline > $OUT/c1.json 2> $OUT/c1.err; echo "c1 rc=$?"; python -c "
import json; d=json.loads(open('$OUT/c1.json').read().splitlines()[-1]); print('C1', d['config']['solve_ms'], 'ms', d['config']['iters_per_solve'], 'it', d['clocks'], 'launches', d['gpu_launches'])"
