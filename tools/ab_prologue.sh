#!/bin/bash
# A/B prologue variants: tools/ab_prologue.sh "label|ENV=.." ...  (bench value + prologue_ms)
for spec in "$@"; do
  label=${spec%%|*}; envs=${spec#*|}
  env $envs timeout 300 python bench.py --steps 60 --warmup 3 --no-cpu-baseline --parity-envs 0 > gpurun_out/abpro_$label.log 2>&1
  echo "$label $(grep -o '"value": [0-9.e+]*' gpurun_out/abpro_$label.log | head -1) $(grep -o '"prologue_ms": [0-9.e+]*' gpurun_out/abpro_$label.log)"
done
