#!/bin/bash
# Round-2 GPU call J: ncu of the stream V-cycle kernel at cfg3 levels 3 and 5.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:merge_stream -s 2 -c 1 \
    -o gpurun_out/stream_L3 python tools/vcycle_levels.py 3 1 > gpurun_out/ncu_stream_L3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:merge_stream -s 4 -c 1 \
    -o gpurun_out/stream_L5 python tools/vcycle_levels.py 3 1 > gpurun_out/ncu_stream_L5.log 2>&1
tail -2 gpurun_out/ncu_stream_L3.log gpurun_out/ncu_stream_L5.log
