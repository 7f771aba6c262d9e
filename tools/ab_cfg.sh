#!/bin/bash
# A/B kernel variants on one bench config: tools/ab_cfg.sh TAG CONFIG "label|ENV=.." ...
TAG=$1; CFG=$2; shift 2
OUT=gpurun_out/$TAG; mkdir -p $OUT
for spec in "$@"; do
  label=${spec%%|*}; envs=${spec#*|}
  env $envs timeout 300 python bench.py --config $CFG --steps 40 --warmup 3 --no-cpu-baseline --parity-envs 0 > $OUT/$CFG-$label.log 2>&1
  v=$(grep -o '"value": [0-9.e+]*' $OUT/$CFG-$label.log | head -1)
  k=$(grep -o '"kernel_ms": [0-9.e+]*' $OUT/$CFG-$label.log | head -1)
  echo "$CFG $label $v $k" | tee -a $OUT/summary.txt
done
