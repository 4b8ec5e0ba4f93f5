#!/bin/bash
# Round-2 GPU call N: ncu of the wide V-cycle kernel (cfg3 levels 10 and 13, down).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:merge_wide -s 4 -c 1 \
    -o gpurun_out/wide_L13 python tools/vcycle_levels.py 3 1 > gpurun_out/ncu_wide_L13.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:merge_wide -s 1 -c 1 \
    -o gpurun_out/wide_L10 python tools/vcycle_levels.py 3 1 > gpurun_out/ncu_wide_L10.log 2>&1
tail -n 2 gpurun_out/ncu_wide_L13.log
