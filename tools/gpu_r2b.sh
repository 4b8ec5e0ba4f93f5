#!/bin/bash
# Round-2 GPU call B: cfg3 golden (box host, background), full GPU test suite.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/golden
( ulimit -v 185000000; timeout 3000 python tools/make_golden.py --config 3 --threads 16 \
    --out gpurun_out/golden > gpurun_out/golden3.log 2>&1; echo "golden rc=$?" >> gpurun_out/golden3.log ) &
GOLD=$!
( while kill -0 $GOLD 2>/dev/null; do free -g | sed -n 2p >> gpurun_out/golden3_mem.log; sleep 20; done ) &
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rf \
    > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
wait $GOLD
tail -15 gpurun_out/pytest_gpu.log; tail -4 gpurun_out/golden3.log; tail -3 gpurun_out/golden3_mem.log
