#!/bin/bash
# Refresh the measured numbers committed under profiles/ (run under gpurun on one B200):
#   benches for every config, the ncu launch list of the default bench command, and an
#   ncu --set full capture of the render kernel (configs 2, 5, 3 and paper).
#   tools/refresh_profiles.sh TAG
TAG=${1:-refresh}
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python bench.py > $OUT/bench_cfg2.log 2>&1; echo "rc=$?" >> $OUT/bench_cfg2.log
for c in cfg3 cfg5 cfg5_1m paper; do
  timeout 900 python bench.py --config $c --steps 60 > $OUT/bench_$c.log 2>&1; echo "rc=$?" >> $OUT/bench_$c.log
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/reference_arm.log 2>&1
# launch list (per-launch times are cold-cache and serialised: compare shares only)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file $OUT/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch.log 2>&1
for c in cfg2 cfg5 cfg3 paper; do
  timeout 300 python tools/profile_step.py --config $c --steps 3 > $OUT/prof_plain_$c.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:render_kernel -s 1 -c 1 \
     -o $OUT/prof_render_$c python tools/profile_step.py --config $c --steps 3 > $OUT/ncu_$c.log 2>&1
  echo "ncu_rc=$?" >> $OUT/ncu_$c.log
done
grep -ho '"value": [0-9.e+]*' $OUT/bench_*.log | head -20
