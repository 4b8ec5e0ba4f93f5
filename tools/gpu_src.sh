#!/bin/bash
# Source-level stall samples of one kernel: ncu --set full --import-source, then the source page as CSV.
# usage: gpu_src.sh <kernel regex> <launch skip> <name> <command...>
cd "$GRAFT_REPO_ROOT"; O=gpurun_out/src; mkdir -p $O
k=$1; s=$2; n=$3; shift 3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c 1 -o $O/$n "$@" > $O/$n.log 2>&1
ncu -i $O/$n.ncu-rep --page source --csv > $O/${n}_source.csv 2>/dev/null
python tools/ncu_full_summary.py $O/$n.ncu-rep "$k" | tail -n +3 | head -24
rm -f $O/$n.ncu-rep
