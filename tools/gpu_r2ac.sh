#!/bin/bash
# Round-2 GPU call AC: V-cycle level profiles at cfg2 and cfg1, and the cfg2 bench kernel split.
cd "$GRAFT_REPO_ROOT"
for c in 2 1; do HPSB_PROFILE_LEVELS=1 timeout 300 python tools/vcycle_levels.py $c 5 2>&1 | grep -v "Exception\|Traceback\|File \|AttributeError"; done
timeout 900 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg2_ac.json 2> gpurun_out/bench_cfg2_ac.err
python -c "
import json; d=json.load(open('gpurun_out/bench_cfg2_ac.json'))
print(d['value'], d['solve_ms_per_step'], d['roofline_gmres']['frac'], d['iterations'], d['setup'])
print({k: v for k, v in d['kernels'].items() if v['ms'] > 0.5})"
