#!/bin/bash
# GPU check at HEAD: the GPU suite, then the default (cfg3) bench line.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rf \
    > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
echo "bench rc=$?" >> gpurun_out/bench_cfg3.err
tail -3 gpurun_out/pytest_gpu.log; head -c 1500 gpurun_out/bench_cfg3.json
