#!/bin/bash
# Element-stage launch list: cfg3 element probe under ncu (time + DRAM bytes per launch), summarised by kernel.
cd "$GRAFT_REPO_ROOT"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/el_launches.csv python tools/element_probe.py 3 2 > gpurun_out/el_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/el_launches.csv "element probe cfg3 (2 builds)" | tee gpurun_out/el_launches.txt
