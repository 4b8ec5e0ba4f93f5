#!/bin/bash
# One-shot environment probe on the GPU box (Eigen presence, cores, CPU model, GPU).
mkdir -p gpurun_out
{
  echo "== nproc: $(nproc)"; lscpu | grep -E "Model name|Socket|Thread|Core" ; free -g | head -2
  echo "== eigen:"; find / -xdev \( -name "Eigen" -o -name "eigen3" \) -maxdepth 6 -type d 2>/dev/null | head
  nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
  ./tools/fp64_peak
} > gpurun_out/probe.log 2>&1
cat gpurun_out/probe.log
