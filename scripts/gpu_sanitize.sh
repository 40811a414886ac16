#!/bin/bash
# One compute-sanitizer tool per gpurun call (B200_PROFILING.md): TOOL=memcheck|racecheck|synccheck|initcheck
OUT=gpurun_out/${TAG:-san}; mkdir -p $OUT
TOOL=${TOOL:-memcheck}
python scripts/sanitize_paths.py > $OUT/plain_$TOOL.log 2>&1; rc=$?; echo "plain rc=$rc"
[ $rc -eq 0 ] || exit 1
timeout 2400 compute-sanitizer --tool $TOOL --print-limit 20 ${SAN_ARGS} python scripts/sanitize_paths.py > $OUT/san_$TOOL.log 2>&1
echo "sanitizer $TOOL rc=$?"
grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Error|error" $OUT/san_$TOOL.log | tail -5
