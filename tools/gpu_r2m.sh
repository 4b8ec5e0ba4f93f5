#!/bin/bash
# Round-2 GPU call M: V-cycle level profile (cfg3) + quick parity subset.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
HPSB_PROFILE_LEVELS=1 timeout 600 python tools/vcycle_levels.py 3 5 > gpurun_out/vlevels_cfg3_m.txt 2>&1
head -12 gpurun_out/vlevels_cfg3_m.txt
timeout 900 python -m pytest tests/test_gpu_golden.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "precond or fgmres or golden" 2>&1 | tail -2
