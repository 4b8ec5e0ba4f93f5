#!/bin/bash
# Round-2 GPU call L: stream levels (late PDL trigger, >= 96 KB merges):
# GPU suite, cfg3 bench, V-cycle level profile, ncu of the level-2 stream step.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rf \
    > gpurun_out/pytest_gpu_l.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_l.log
tail -4 gpurun_out/pytest_gpu_l.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_cfg3_l.json 2> gpurun_out/bench_cfg3_l.err
python -c "
import json; d=json.load(open('gpurun_out/bench_cfg3_l.json'))
print({k: d[k] for k in ['value','setup','solve_ms_per_step','roofline_setup','roofline_gmres','iterations','e2e']})"
HPSB_PROFILE_LEVELS=1 timeout 600 python tools/vcycle_levels.py 3 5 > gpurun_out/vlevels_cfg3_l.txt 2>&1
head -30 gpurun_out/vlevels_cfg3_l.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:merge_stream -s 0 -c 1 \
    -o gpurun_out/stream_L2 python tools/vcycle_levels.py 3 1 > gpurun_out/ncu_stream_L2.log 2>&1
tail -1 gpurun_out/ncu_stream_L2.log
