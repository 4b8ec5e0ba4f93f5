#!/bin/bash
# Multi-RHS path check: multi-RHS / sharded / golden parity tests, the per-level 16-RHS apply profile at cfg4, the cfg4 bench.
cd "$GRAFT_REPO_ROOT"
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "rhs or batch or multi or cfg4 or golden" 2>&1 | tail -3
HPSB_PROFILE_LEVELS=1 timeout 600 python tools/vcycle_levels_batch.py 4 16 3 2>&1 | grep -v "Exception\|Traceback\|File\|Attribute" | head -8
timeout 1500 python bench.py --config 4 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']
print('cfg4 value %.3e' % d['value'], 'solve ms', round(d['solve_ms_per_step'],1), 'block its', d['roofline_gmres'].get('block_iterations'), {n: round(k[n]['ms'],1) for n in ('vcycle_up_batch','vcycle_down_batch','gmres_orth','skeleton_matvec_batch','coarse_matvec_batch') if n in k})"
