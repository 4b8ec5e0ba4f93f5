#!/bin/bash
# ncu --set full of the element diag / dinv kernels (cfg3 element probe).
cd "$GRAFT_REPO_ROOT"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"v5_diag|v5_dinv" \
  --launch-skip 12 -c 2 -o gpurun_out/el_diag python tools/element_probe.py 3 2 > gpurun_out/el_diag.log 2>&1
python tools/ncu_full_summary.py gpurun_out/el_diag.ncu-rep "element diag kernels cfg3" | tee gpurun_out/el_diag.txt | head -60
ncu -i gpurun_out/el_diag.ncu-rep --page source --csv --kernel-name regex:v5_diag > gpurun_out/el_diag_source.csv 2>/dev/null
