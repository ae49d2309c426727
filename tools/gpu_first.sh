#!/bin/bash
# first GPU smoke: stage-by-stage numerics of every config, each in its own process
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/gpu.txt 2>&1
for c in "c4 4" "c1" "c2_bf16 4" "c3 4" "c2_f32 4" "c2_bf16" "c3" "c4" "c2_f32"; do
  tag=${c// /_}
  timeout 180 python tools/gpu_debug.py $c > gpurun_out/dbg_$tag.log 2>&1
  echo "$c exit $?" | tee -a gpurun_out/summary.txt
done
cat gpurun_out/dbg_*.log
