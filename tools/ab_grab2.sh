#!/bin/bash
# A/B: tile batches in registers (MDRT_GRAB_REG) vs shared memory with carveout 0
for c in cfg2 cfg3 paper cfg5; do
  bash tools/ab_cfg.sh grab2 $c "g1|MDRT_LIB=build/libmdrt_g1.so" "r2|MDRT_LIB=build/libmdrt_r2.so" "r4|MDRT_LIB=build/libmdrt_r4.so" "g4c0|MDRT_LIB=build/libmdrt_g4.so MDRT_CARVEOUT=0"
done
