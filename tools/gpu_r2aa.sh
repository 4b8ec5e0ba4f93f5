#!/bin/bash
# Round-2 GPU call AA: multi-RHS parity + cfg4 bench (batched TMA-streamed CGS2).
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "batch or multi_rhs or cfg4 or sharded" 2>&1 | tail -2
timeout 1200 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4_aa.json 2> gpurun_out/bench_cfg4_aa.err
python -c "
import json; d=json.load(open('gpurun_out/bench_cfg4_aa.json'))
print(d['value'], d['solve_ms_per_step'], d['roofline_gmres']['frac'], d['iterations'], d['setup'])
print({k: v for k, v in d['kernels'].items() if v['ms'] > 5})"
