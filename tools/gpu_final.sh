#!/bin/bash
# Round-end rehearsal: smoke(), the reference arm and the default bench as the driver runs them.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/final
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
( time timeout 1700 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/final/bench_reference_cfg3.json 2> gpurun_out/final/bench_reference.err ) 2>&1 | grep real
( time timeout 900 python bench.py > gpurun_out/final/bench_default.json 2> gpurun_out/final/bench_default.err ) 2>&1 | grep real
head -c 700 gpurun_out/final/bench_reference_cfg3.json; echo; head -c 300 gpurun_out/final/bench_default.json
