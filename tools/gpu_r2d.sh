#!/bin/bash
# Round-2 GPU call D: full GPU suite (new sharded data plane, cfg4 golden),
# cfg3 bench with setup trace, cfg3 reference arm.
cd "$GRAFT_REPO_ROOT"
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 -rf \
    > gpurun_out/pytest_gpu_d.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_d.log
HPSB_TRACE=1 HPSB_BENCH_VERBOSE=1 timeout 900 python bench.py --steps 5 --warmup 3 \
    > gpurun_out/bench_cfg3_d.json 2> gpurun_out/bench_cfg3_d.err
echo "bench rc=$?" >> gpurun_out/bench_cfg3_d.err
( ulimit -v 185000000; timeout 1500 python bench.py --impl reference --steps 3 --warmup 1 \
    > gpurun_out/bench_ref_cfg3.json 2> gpurun_out/bench_ref_cfg3.err; echo "ref rc=$?" >> gpurun_out/bench_ref_cfg3.err )
tail -12 gpurun_out/pytest_gpu_d.log; head -c 400 gpurun_out/bench_cfg3_d.json; echo; cat gpurun_out/bench_ref_cfg3.json | head -c 1500; tail -3 gpurun_out/bench_ref_cfg3.err
