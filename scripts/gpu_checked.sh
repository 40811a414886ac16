#!/bin/bash
# The -m gpu suite and every device path against the bounds-checked library
# (_lib_chk/libamgb.so: device asserts on gathers and TMA stage ranges)
OUT=gpurun_out/${TAG:-checked}; mkdir -p $OUT
export AMGB_LIB_PATH=$PWD/paper_1811_05704_b200/_lib_chk/libamgb.so
python -c "import paper_1811_05704_b200 as a; print(a.LIB_PATH)" > $OUT/which.txt
timeout 2400 python -m pytest tests -q -m gpu -rf -p no:randomly > $OUT/tests.log 2>&1; echo "checked tests rc=$?"; tail -2 $OUT/tests.log; grep -E "FAILED|cudaErrorAssert|device-side assert" $OUT/tests.log | head
timeout 900 python scripts/sanitize_paths.py > $OUT/paths.log 2>&1; echo "checked paths rc=$?"; tail -3 $OUT/paths.log
