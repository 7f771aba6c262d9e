#!/bin/bash
# One GPU iteration: parity tests, a short bench, optionally an ncu capture of the render kernel.
#   tools/gpu_check.sh TAG [ncu] [bench-args...]
TAG=${1:-run}; shift
NCU=0
if [ "$1" == "ncu" ]; then NCU=1; shift; fi
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 600 python -m pytest tests -m gpu -q -rA -x > $OUT/pytest_gpu.log 2>&1; echo "pytest_rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python bench.py --steps 100 --no-cpu-baseline "$@" > $OUT/bench.log 2>&1; echo "bench_rc=$?" >> $OUT/bench.log
if [ $NCU == 1 ]; then
  timeout 300 python tools/profile_step.py --steps 3 > $OUT/prof_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:render_kernel -s 1 -c 1 \
     -o $OUT/prof_render python tools/profile_step.py --steps 3 > $OUT/ncu.log 2>&1
  echo "ncu_rc=$?" >> $OUT/ncu.log
fi
tail -n 2 $OUT/pytest_gpu.log; grep -o '"value": [0-9.e+]*' $OUT/bench.log | head -2
