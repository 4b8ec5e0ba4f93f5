#!/bin/bash
# Round-2 GPU call S: ncu evidence for the round-2 kernels at cfg3 -- launch list
# of one bench step (time + DRAM bytes per launch) and --set full captures of
# merge_stream (level 4), merge_wide (level 10), v5_iti_dmma, inverse_dmma, zgemm.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -c 4000 --csv --log-file gpurun_out/launches_cfg3_s.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_bench_s.log 2>&1
tail -n 1 gpurun_out/ncu_bench_s.log
cap() { timeout 600 ncu --set full --clock-control none --import-source on -k regex:$1 -s $2 -c 1 \
    -o gpurun_out/$3 python tools/vcycle_levels.py 3 1 > gpurun_out/ncu_$3.log 2>&1; tail -n 1 gpurun_out/ncu_$3.log; }
cap merge_stream 3 r02_stream_L4
cap merge_wide 1 r02_wide_L10
cap v5_iti_dmma 0 r02_iti_dmma
cap inverse_dmma 20 r02_inverse_dmma
cap zgemm_grouped 40 r02_zgemm
