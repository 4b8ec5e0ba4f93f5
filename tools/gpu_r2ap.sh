#!/bin/bash
# Round-2 GPU call AP: contract checks -- torchrun launcher (1 rank) and the reference arm.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_torchrun.json 2> gpurun_out/bench_torchrun.err
echo "torchrun rc=$?"; tail -c 400 gpurun_out/bench_torchrun.json
( ulimit -v 185000000; timeout 1500 python bench.py --impl reference --steps 3 --warmup 1 \
    > gpurun_out/bench_ref_cfg3_ap.json 2> gpurun_out/bench_ref_cfg3_ap.err; echo "ref rc=$?" )
head -c 600 gpurun_out/bench_ref_cfg3_ap.json
