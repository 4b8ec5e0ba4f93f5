#!/bin/bash
# Round-2 GPU call G (re-entry): sustained FP64 DMMA peak with clocks, full
# GPU suite at HEAD, cfg3 bench, ncu launch list of a short cfg3 bench.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks_throttle_reasons.active,power.draw \
    --format=csv,noheader,nounits -lms 250 > gpurun_out/fp64_clocks.csv &
SMI=$!
./tools/fp64_peak 4 > gpurun_out/fp64_sustained.json
kill $SMI
python - <<'PY'
import json, statistics
d = json.load(open("gpurun_out/fp64_sustained.json"))
rows = [r.split(",") for r in open("gpurun_out/fp64_clocks.csv").read().strip().splitlines()]
sm = [float(r[0]) for r in rows if r[0].strip().isdigit()]
busy = [s for s in sm if s > 500]
d["clocks"] = {"sm_mhz_median": statistics.median(busy or sm), "sm_max_mhz": float(rows[0][1]),
               "reasons": sorted({r[2].strip() for r in rows}), "samples": len(rows),
               "power_w_max": max(float(r[3]) for r in rows)}
d["how"] = "tools/fp64_peak.cu: mma.sync m8n8k4 f64 chains, grid 4x148 x 256 threads, back to back for 4 s, one CUDA-event pair"
json.dump(d, open("gpurun_out/r02_fp64_peak.json", "w"), indent=1)
print(d)
PY
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rf --durations=25 \
    > gpurun_out/pytest_gpu_g.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_g.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_cfg3_g.json 2> gpurun_out/bench_cfg3_g.err
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -c 3000 --csv --log-file gpurun_out/launches_cfg3_g.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_bench_g.log 2>&1
tail -40 gpurun_out/pytest_gpu_g.log
python -c "
import json; d=json.load(open('gpurun_out/bench_cfg3_g.json'))
print({k: d[k] for k in ['value','setup','solve_ms_per_step','roofline_setup','roofline_gmres','roofline','e2e','iterations','clocks']})"
tail -3 gpurun_out/ncu_bench_g.log
