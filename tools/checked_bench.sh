#!/usr/bin/env bash
# Every bench configuration at full size under the bounds-checked build
# (libmdrt_checked.so, MDRT_CHECKS): a check that fails prints MDRT_CHECK and
# aborts the launch. Timings from this build are not bench numbers.
#   gpurun -- 'bash tools/checked_bench.sh'
set -u
mkdir -p gpurun_out/checked
lib=$(python -m paper_2602_03002_b200.build --checked)
rc_all=0
for cfg in cfg2 cfg3 cfg5 cfg5_1m paper; do
    MDRT_LIB=$lib timeout 600 python bench.py --config "$cfg" --steps 3 --warmup 3 --no-cpu-baseline \
        > "gpurun_out/checked/$cfg.log" 2>&1
    rc=$?
    n=$(grep -c MDRT_CHECK "gpurun_out/checked/$cfg.log")
    echo "$cfg rc=$rc checks_failed=$n"
    [ "$rc" -ne 0 ] || [ "$n" -ne 0 ] && rc_all=1
done
exit $rc_all
