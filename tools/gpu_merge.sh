#!/bin/bash
# Merge-stage check: hierarchy / golden / sharded parity tests, then the cfg3 bench kernel table.
cd "$GRAFT_REPO_ROOT"
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -2
for i in 1 2; do
timeout 900 python bench.py --steps 4 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']
print('setup ms', round(d['setup']['ms_per_step'],2), 'solve ms', round(d['solve_ms_per_step'],2), d['iterations'][0], 'setup frac', round(d['roofline_setup']['frac'],4), 'zgemm frac', round(d['roofline']['frac'],4))
print({n: k[n]['ms'] for n in ('zgemm_dmma','merge_copy','element_iti','zinverse_smem') if n in k})"
done
