#!/bin/bash
# Round-2 GPU call AH: ncu evidence refresh -- cfg3 launch list of one bench step and
# --set full captures of orth_stream, gemv_stream (interface matvec), coarse_wide.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -c 4000 --csv --log-file gpurun_out/launches_cfg3_ah.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_bench_ah.log 2>&1
tail -n 1 gpurun_out/ncu_bench_ah.log
cap() { timeout 900 ncu --set full --clock-control none --import-source on -k regex:$1 -s $2 -c 1 \
    -o gpurun_out/$3 python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_$3.log 2>&1; tail -n 1 gpurun_out/ncu_$3.log; }
cap orth_stream 60 r02_orth_stream
cap gemv_stream 20 r02_gemv_stream
cap coarse_wide 10 r02_coarse_wide
