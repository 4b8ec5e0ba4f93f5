#!/bin/bash
# Round-2 GPU call R: merge GEMM variant timing (setup probe under per-kernel events) + merge parity.
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -m gpu -q -p no:cacheprovider -x -k "hierarchy or level or merge" 2>&1 | tail -2
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg3_r.json 2> gpurun_out/bench_cfg3_r.err
python -c "
import json; d=json.load(open('gpurun_out/bench_cfg3_r.json'))
print(d['setup'], d['roofline_setup']['frac'])
print({k: v for k, v in d['kernels'].items() if v['ms'] > 3})"
