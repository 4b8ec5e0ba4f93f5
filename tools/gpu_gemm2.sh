#!/bin/bash
# ncu --set full of two large merge GEMM launches (cfg3 setup probe, levels 12-13).
cd "$GRAFT_REPO_ROOT"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:zgemm_grouped \
  --launch-skip 270 -c 2 -o gpurun_out/zgemm_big python tools/setup_probe.py 3 1 > gpurun_out/zgemm_big.log 2>&1
python tools/ncu_full_summary.py gpurun_out/zgemm_big.ncu-rep "zgemm_grouped, cfg3 level 13" | tee gpurun_out/zgemm_big.txt | head -60
ncu -i gpurun_out/zgemm_big.ncu-rep --page source --csv > gpurun_out/zgemm_big_source.csv 2>/dev/null
