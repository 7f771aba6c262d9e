#!/bin/bash
# Envs per GPU at the config-2 shape: bench lines for 512 ... 32768 envs (one B200).
#   gpurun -- 'bash tools/batch_scaling.sh'   ->  gpurun_out/batch_scaling.jsonl
mkdir -p gpurun_out; : > gpurun_out/batch_scaling.jsonl
for n in 512 1024 2048 4096 8192 16384 32768; do
  timeout 600 python bench.py --envs $n --steps 40 --no-cpu-baseline 2>/dev/null | grep '^{' >> gpurun_out/batch_scaling.jsonl
done
