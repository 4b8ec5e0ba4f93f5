#!/bin/bash
# Round-2 GPU call I: warp-per-merge TMA-ring V-cycle levels (vcycle_stream.cu)
# + DMMA Gauss-Jordan: GPU suite, V-cycle level profile, cfg3 bench, ncu of the
# stream kernel.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
HPSB_PROFILE_LEVELS=1 timeout 600 python tools/vcycle_levels.py 3 5 > gpurun_out/vlevels_cfg3_i.txt 2>&1
head -40 gpurun_out/vlevels_cfg3_i.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rf \
    > gpurun_out/pytest_gpu_i.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_i.log
tail -25 gpurun_out/pytest_gpu_i.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_cfg3_i.json 2> gpurun_out/bench_cfg3_i.err
python -c "
import json; d=json.load(open('gpurun_out/bench_cfg3_i.json'))
print({k: d[k] for k in ['value','setup','solve_ms_per_step','roofline_setup','roofline_gmres','iterations']})
print({k: v for k, v in d['kernels'].items() if v['ms'] > 1})"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:merge_stream -s 2 -c 1 \
    -o gpurun_out/stream_cfg3 python tools/vcycle_levels.py 3 1 > gpurun_out/ncu_stream_i.log 2>&1
tail -3 gpurun_out/ncu_stream_i.log
