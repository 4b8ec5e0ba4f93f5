#!/bin/bash
# Host/device overlap of the setup: bench steps with the per-phase wall clock (HPSB_BENCH_VERBOSE) and one traced build (HPSB_TRACE).
cd "$GRAFT_REPO_ROOT"
HPSB_BENCH_VERBOSE=1 timeout 900 python bench.py --steps 6 --warmup 3 --no-cpu-baseline 2>&1 >/dev/null | grep "setup wall" 
HPSB_BENCH_VERBOSE=1 timeout 900 python bench.py --steps 6 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('setup ms', round(d['setup']['ms_per_step'],2))"
HPSB_TRACE=1 timeout 600 python tools/setup_probe.py 3 2 2>&1 | grep -v "^\[gemm\]" | tail -60
