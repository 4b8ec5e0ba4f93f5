#!/bin/bash
# Round-2 GPU call A: cfg3 golden generation on the box host (background),
# GPU tests, sustained FP64 probe, cfg3 bench.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/golden
nproc > gpurun_out/nproc.txt; free -g >> gpurun_out/nproc.txt
( ulimit -v 170000000; timeout 3000 python tools/make_golden.py --config 3 --threads 16 \
    --out gpurun_out/golden > gpurun_out/golden3.log 2>&1 ) &
GOLD=$!
# sustained FP64 with clocks sampled
( nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active \
    --format=csv,noheader,nounits -lms 200 > gpurun_out/fp64_clocks.csv 2>&1 & SMI=$!;
  timeout 120 ./tools/fp64_peak 4 > gpurun_out/fp64_sustained.json 2>&1; kill $SMI )
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rf \
    > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
echo "bench rc=$?" >> gpurun_out/bench_cfg3.err
wait $GOLD
echo "golden rc=$?" >> gpurun_out/golden3.log
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/golden3.log; head -c 600 gpurun_out/bench_cfg3.json
