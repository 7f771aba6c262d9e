#!/bin/bash
# Round-2 refresh of the measured numbers under profiles/ (run under gpurun on one B200):
#   GPU test suite, benches for every config, the live-reference arm, the ncu launch
#   list of the default bench command and ncu --set full captures of the render kernel.
#   tools/refresh_r02.sh TAG [skip-tests]
TAG=${1:-r02}
OUT=gpurun_out/$TAG; mkdir -p $OUT
if [ "$2" != "skip-tests" ]; then
  timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
  tail -3 $OUT/pytest_gpu.log
fi
timeout 900 python bench.py --steps 100 --warmup 5 > $OUT/bench_cfg2.log 2>&1; echo "rc=$?" >> $OUT/bench_cfg2.log
for c in cfg3 cfg5 cfg5_1m paper; do
  timeout 900 python bench.py --config $c --steps 40 --warmup 5 > $OUT/bench_$c.log 2>&1; echo "rc=$?" >> $OUT/bench_$c.log
done
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $OUT/reference_arm.log 2>&1; echo "rc=$?" >> $OUT/reference_arm.log
# launch list (per-launch times are cold-cache and serialised: compare shares only)
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --parity-envs 0 > $OUT/plain_launch.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file $OUT/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --parity-envs 0 > $OUT/ncu_launch.log 2>&1
for c in cfg2 cfg5; do
  timeout 300 python tools/profile_step.py --config $c --steps 3 > $OUT/prof_plain_$c.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:render_kernel -s 1 -c 1 \
     -o $OUT/prof_render_$c python tools/profile_step.py --config $c --steps 3 > $OUT/ncu_$c.log 2>&1
  echo "ncu_rc=$?" >> $OUT/ncu_$c.log
done
grep -ho '"value": [0-9.e+]*' $OUT/bench_*.log | head -20
