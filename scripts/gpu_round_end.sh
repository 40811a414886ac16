#!/bin/bash
# Round-end evidence in one call: the checked-build GPU suite, then the final evidence
# (tests, smoke, bench + reference arm, configs, ncu launch list + --set full)
TAG=${TAG:-r2_end} bash scripts/gpu_checked.sh
TAG=${TAG2:-r2_final3} bash scripts/gpu_final_r2.sh
