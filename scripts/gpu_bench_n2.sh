#!/bin/bash
# bench.py's N > 1 path end to end on a one-GPU box (TEST ONLY: AMGB_BENCH_ONE_GPU=1 puts
# every rank on GPU 0 with gloo + the shm transport): strong 2 ranks at 128^3, weak 2 ranks
OUT=gpurun_out/${TAG:-n2}; mkdir -p $OUT
export AMGB_BENCH_ONE_GPU=1 AMGB_NCCL_TIMEOUT_S=300
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --steps 3 --warmup 3 --size 128 > $OUT/strong2.log 2>&1; echo "strong2 rc=$?"; grep '"metric"' $OUT/strong2.log | head -c 900; echo
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 \
  bench.py --gpus 2 --steps 3 --warmup 3 --size 96 --scaling weak > $OUT/weak2.log 2>&1; echo "weak2 rc=$?"; grep '"metric"' $OUT/weak2.log | head -c 900; echo
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29535 \
  bench.py --gpus 2 --impl reference --steps 2 --warmup 1 --size 64 > $OUT/ref2.log 2>&1; echo "ref2 rc=$?"; tail -c 300 $OUT/ref2.log
unset AMGB_BENCH_ONE_GPU
timeout 900 python scripts/ab_inproc.py --n 256 --rounds 4 --solves 3 --variants "minb4:|;minb5:AMGB_TMA_MINB=5|" > $OUT/ab_minb5.txt 2>&1; echo "ab rc=$?"; tail -2 $OUT/ab_minb5.txt
