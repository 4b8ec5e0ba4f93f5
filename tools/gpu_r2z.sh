#!/bin/bash
# Round-2 GPU call Z: determinism probes, GPU suite, cfg3 bench (proxy-fenced TMA consumers).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 600 python tools/orth_probe.py 3 4 40 2>&1 | grep "spread"
timeout 600 python tools/determinism_probe.py 3 4 2>&1 | grep "iterations\|solution\|MG"
timeout 600 python tools/determinism_probe.py 2 4 2>&1 | grep "iterations\|solution\|MG"
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rf > gpurun_out/pytest_gpu_z.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_z.log
tail -3 gpurun_out/pytest_gpu_z.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_cfg3_z.json 2> gpurun_out/bench_cfg3_z.err
python -c "
import json; d=json.load(open('gpurun_out/bench_cfg3_z.json'))
print(d['value'], d['solve_ms_per_step'], d['roofline_gmres']['frac'], d['iterations'], d['setup'], d['e2e']['value'])
print({k: v for k, v in d['kernels'].items() if v['ms'] > 3})"
HPSB_PROFILE_LEVELS=1 timeout 600 python tools/vcycle_levels.py 3 5 2>&1 | grep -v "Exception\|Traceback\|File \|AttributeError" > gpurun_out/vlevels_cfg3_z.txt
head -3 gpurun_out/vlevels_cfg3_z.txt
