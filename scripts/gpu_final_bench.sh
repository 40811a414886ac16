#!/bin/bash
# bench-only final evidence (tests already run on this build): box identity, bench + reference
# arm, configs, ncu launch list + --set full (scripts/gpu_final_r2.sh with SKIP_TESTS)
OUT=gpurun_out/${TAG:-r2_final7}; mkdir -p $OUT
nvidia-smi --query-gpu=name,serial,pci.bus_id,clocks.max.sm,clocks.max.mem,memory.total,power.limit --format=csv > $OUT/box.txt 2>&1; cat $OUT/box.txt
SKIP_TESTS=1 TAG=${TAG:-r2_final7} bash scripts/gpu_final_r2.sh
