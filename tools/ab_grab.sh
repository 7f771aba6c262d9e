#!/bin/bash
# A/B: shared-pool tiles taken 1/2/4 per atomic (MDRT_GRAB builds in build/), two interleaved rounds
for r in 1 2; do
  for c in cfg2 cfg3 paper cfg5; do
    bash tools/ab_cfg.sh grab_r$r $c "g1|MDRT_LIB=build/libmdrt_g1.so" "g2|MDRT_LIB=build/libmdrt_g2.so" "g4|MDRT_LIB=build/libmdrt_g4.so"
  done
done
