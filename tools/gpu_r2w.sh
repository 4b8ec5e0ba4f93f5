#!/bin/bash
# Round-2 GPU call W: Krylov parity subset + cfg3 bench (orth through the TMA-streamed kernel).
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_golden.py tests/test_gpu_parity.py tests/test_gpu_boundary.py -m gpu -q -p no:cacheprovider -x -k "fgmres or gmres or orth or solve or history or report" 2>&1 | tail -2
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg3_w.json 2> gpurun_out/bench_cfg3_w.err
python -c "
import json; d=json.load(open('gpurun_out/bench_cfg3_w.json'))
print(d['value'], d['solve_ms_per_step'], d['roofline_gmres']['frac'], d['iterations'])
print({k: v for k, v in d['kernels'].items() if v['ms'] > 3})"
