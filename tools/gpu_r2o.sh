#!/bin/bash
# Round-2 GPU call O: GPU suite, cfg3 bench, V-cycle level profile.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rf \
    > gpurun_out/pytest_gpu_o.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_o.log
tail -4 gpurun_out/pytest_gpu_o.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_cfg3_o.json 2> gpurun_out/bench_cfg3_o.err
python -c "
import json; d=json.load(open('gpurun_out/bench_cfg3_o.json'))
print({k: d[k] for k in ['value','setup','solve_ms_per_step','roofline_setup','roofline_gmres','iterations','e2e']})"
HPSB_PROFILE_LEVELS=1 timeout 600 python tools/vcycle_levels.py 3 5 > gpurun_out/vlevels_cfg3_o.txt 2>&1
grep -v "Exception\|Traceback\|File \|AttributeError" gpurun_out/vlevels_cfg3_o.txt
