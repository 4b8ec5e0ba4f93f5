#!/bin/bash
# Round-2 GPU call AE: GPU suite + bench lines cfg1-4 (+ cfg3 reference arm sample kept from earlier).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rf > gpurun_out/pytest_gpu_ae.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_ae.log
tail -3 gpurun_out/pytest_gpu_ae.log
for c in 3 2 1 4; do
  timeout 1200 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_cfg${c}_ae.json 2> gpurun_out/bench_cfg${c}_ae.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_cfg${c}_ae.json'))
print('cfg$c', d['value'], d['solve_ms_per_step'], d['roofline_gmres']['frac'], d['iterations'][0], d['setup']['value'], d['roofline_setup']['frac'], d['e2e']['value'])"
done
