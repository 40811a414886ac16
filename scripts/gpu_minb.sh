#!/bin/bash
OUT=gpurun_out/${TAG:-minb}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_formats.py -q -m gpu -x -k "vcycle_and_solve or value_indexed" > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -1 $OUT/tests.log
timeout 1200 python scripts/ab_inproc.py --n 256 --rounds 4 --solves 3 --variants "base:|;minb3:AMGB_TMA_MINB=3|;vidx:AMGB_VIDX=1|;vidx_minb3:AMGB_VIDX=1,AMGB_TMA_MINB=3|" > $OUT/ab_256.txt 2>&1; echo "ab rc=$?"; tail -4 $OUT/ab_256.txt
