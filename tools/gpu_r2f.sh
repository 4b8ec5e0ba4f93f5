#!/bin/bash
# Round-2 GPU call F: V-cycle per-level profile (cfg3), ncu launch list of a
# short cfg3 bench, one ncu --set full zgemm capture, sharded tests, cfg4 bench.
cd "$GRAFT_REPO_ROOT"
HPSB_PROFILE_LEVELS=1 timeout 600 python tools/vcycle_levels.py 3 5 > gpurun_out/vlevels_cfg3.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_sharded.py -m gpu -q -p no:cacheprovider --timeout 600 -rf \
    > gpurun_out/pytest_sharded_f.log 2>&1
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -c 2500 --csv --log-file gpurun_out/launches_cfg3.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:zgemm_grouped -s 40 -c 1 \
    -o gpurun_out/zgemm_cfg3 python tools/setup_probe.py 3 1 > gpurun_out/ncu_zgemm.log 2>&1
cat gpurun_out/vlevels_cfg3.txt; tail -5 gpurun_out/pytest_sharded_f.log
python -c "
import json; d=json.load(open('gpurun_out/bench_cfg4.json'))
print({k: d[k] for k in ['value','setup','solve_ms_per_step','roofline_setup','roofline_gmres','iterations']})"
tail -3 gpurun_out/ncu_bench.log; tail -3 gpurun_out/ncu_zgemm.log
