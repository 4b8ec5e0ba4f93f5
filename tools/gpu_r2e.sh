#!/bin/bash
# Round-2 GPU call E: sharded multi-RHS diagnostic, sharded tests, cfg3 bench
# (pinned-ring pool), cfg3 reference arm (lean oracle elements).
cd "$GRAFT_REPO_ROOT"
timeout 600 python tools/diag_sharded_batch.py > gpurun_out/diag_sb.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_sharded.py -m gpu -q -p no:cacheprovider --timeout 600 -rf \
    > gpurun_out/pytest_sharded_e.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_cfg3_e.json 2> gpurun_out/bench_cfg3_e.err
( ulimit -v 185000000; timeout 1500 python bench.py --impl reference --steps 3 --warmup 1 \
    > gpurun_out/bench_ref_cfg3.json 2> gpurun_out/bench_ref_cfg3.err; echo "ref rc=$?" >> gpurun_out/bench_ref_cfg3.err )
cat gpurun_out/diag_sb.log; tail -8 gpurun_out/pytest_sharded_e.log
python -c "
import json; d=json.load(open('gpurun_out/bench_cfg3_e.json'))
print({k: d[k] for k in ['value','setup','solve_ms_per_step','roofline_setup','roofline_gmres']})"
head -c 1500 gpurun_out/bench_ref_cfg3.json; tail -3 gpurun_out/bench_ref_cfg3.err
