#!/bin/bash
# Round-2 GPU call H: DMMA blocked Gauss-Jordan (element ItI + merge inverses):
# parity tests, cfg3 bench, setup launch list, ncu of the new kernels, V-cycle
# per-level profile of cfg3.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rf -x \
    > gpurun_out/pytest_gpu_h.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_h.log
tail -15 gpurun_out/pytest_gpu_h.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_cfg3_h.json 2> gpurun_out/bench_cfg3_h.err
python -c "
import json; d=json.load(open('gpurun_out/bench_cfg3_h.json'))
print({k: d[k] for k in ['value','setup','solve_ms_per_step','roofline_setup','roofline_gmres','iterations']})
print({k: v for k, v in d['kernels'].items() if v['ms'] > 1})"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/launches_setup_cfg3_h.csv \
    python tools/setup_probe.py 3 1 > gpurun_out/ncu_setup_h.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:v5_iti_dmma -c 1 \
    -o gpurun_out/iti_dmma_cfg3 python tools/setup_probe.py 3 1 > gpurun_out/ncu_iti_h.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:inverse_dmma -s 20 -c 1 \
    -o gpurun_out/inv_dmma_cfg3 python tools/setup_probe.py 3 1 > gpurun_out/ncu_inv_h.log 2>&1
HPSB_PROFILE_LEVELS=1 timeout 600 python tools/vcycle_levels.py 3 5 > gpurun_out/vlevels_cfg3.txt 2>&1
cat gpurun_out/vlevels_cfg3.txt | head -70
tail -3 gpurun_out/ncu_setup_h.log gpurun_out/ncu_iti_h.log gpurun_out/ncu_inv_h.log
