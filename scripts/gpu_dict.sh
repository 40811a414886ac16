#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || exit 1
timeout 300 python -m pytest tests/test_gpu_dict.py -x -q > $OUT/dicttests.log 2>&1; echo "dict tests rc=$?"; tail -5 $OUT/dicttests.log
AB_VAR=AMGB_NO_DICT bash scripts/gpu_ab_env.sh
BENCH_ARGS="--problem poisson_perm --n 150" AB_VAR=AMGB_NO_DICT bash -c 'for v in 0 1; do if [ $v = 1 ]; then export AMGB_NO_DICT=1; fi; python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e $BENCH_ARGS > gpurun_out/perm_$v.json 2>gpurun_out/perm_$v.err; tail -c 300 gpurun_out/perm_$v.json; done'
