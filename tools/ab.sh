#!/bin/bash
# A/B kernel variants: tools/ab.sh TAG "label|ENV=.. ENV2=.." ...   (runs a short bench per variant)
TAG=$1; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
for spec in "$@"; do
  label=${spec%%|*}; envs=${spec#*|}
  env $envs timeout 300 python bench.py --steps 60 --warmup 3 --no-cpu-baseline --parity-envs 0 > $OUT/$label.log 2>&1
  v=$(grep -o '"value": [0-9.e+]*' $OUT/$label.log | head -1)
  k=$(grep -o '"kernel_ms": [0-9.e+]*' $OUT/$label.log | head -1)
  echo "$label $v $k" | tee -a $OUT/summary.txt
done
