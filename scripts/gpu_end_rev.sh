#!/bin/bash
# round-end evidence of the build without the shared-memory SELL table, with a 2-build A/B first
OUT=gpurun_out/r2ab4; mkdir -p $OUT
nvidia-smi --query-gpu=name,serial,pci.bus_id --format=csv > $OUT/box.txt 2>&1
timeout 300 python scripts/class_times.py --n 256 > $OUT/classes.txt 2>&1; grep -E "unprofiled|transfer|A coarse|A0 pass" $OUT/classes.txt
TAG=r2_end5 TAG2=r2_final8 bash scripts/gpu_round_end.sh
