#!/bin/bash
# Round-2 GPU call AB: element parity + cfg3 setup (diag factorisation fused into the update launch).
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "element or golden or level" 2>&1 | tail -2
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg3_ab.json 2> gpurun_out/bench_cfg3_ab.err
python -c "
import json; d=json.load(open('gpurun_out/bench_cfg3_ab.json'))
print(d['value'], d['setup'], d['roofline_setup']['frac'], d['iterations'])
print({k: v for k, v in d['kernels'].items() if v['ms'] > 5})"
