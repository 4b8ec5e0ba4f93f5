#!/bin/bash
# Round-2 GPU call C: cfg4 golden (first 4 RHS, box host, background); orthogonality
# diagnostic; boundary + full-size golden tests (cfg0-3).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/golden
( ulimit -v 185000000; timeout 3000 python tools/make_golden.py --config 4 --rhs 4 --threads 16 \
    --out gpurun_out/golden > gpurun_out/golden4.log 2>&1; echo "golden rc=$?" >> gpurun_out/golden4.log ) &
GOLD=$!
( while kill -0 $GOLD 2>/dev/null; do free -g | sed -n 2p >> gpurun_out/golden4_mem.log; sleep 20; done ) &
timeout 600 python tools/diag_orth.py > gpurun_out/diag_orth.log 2>&1
timeout 2400 python -m pytest tests/test_gpu_boundary.py tests/test_gpu_golden.py tests/test_gpu_sharded.py -m gpu -q -p no:cacheprovider --timeout 1200 -rf \
    > gpurun_out/pytest_gpu_c.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_c.log
wait $GOLD
cat gpurun_out/diag_orth.log; tail -15 gpurun_out/pytest_gpu_c.log; tail -8 gpurun_out/golden4.log; tail -2 gpurun_out/golden4_mem.log
