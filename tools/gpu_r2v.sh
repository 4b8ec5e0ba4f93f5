#!/bin/bash
# Round-2 GPU call V: GPU suite + ncu --set full of the CGS2 orth kernels (cfg3 bench step).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rf > gpurun_out/pytest_gpu_v.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_v.log
tail -3 gpurun_out/pytest_gpu_v.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:orth_kernel -s 60 -c 2 \
    -o gpurun_out/r02_orth python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_orth.log 2>&1
tail -n 1 gpurun_out/ncu_orth.log
