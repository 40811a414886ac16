OUT=gpurun_out/r2m; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_formats.py tests/test_gpu_fullsize.py tests/test_gpu_dict.py tests/test_gpu_sigma.py tests/test_gpu_batched.py tests/test_gpu_mixed.py tests/test_gpu_dist.py tests/test_gpu_parity.py -q -m gpu -x > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -2 $OUT/tests.log
TAG=r2m ROUNDS=3 bash scripts/gpu_ab_lib.sh
