#!/bin/bash
# full ncu capture of one arm_rate_kernel launch (run under gpurun)
set -e
CMD="python bench.py --images 2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"arm_rate_kernel" -s 3 -c 1 -o gpurun_out/prof_arm $CMD > gpurun_out/ncu_full.log 2>&1
echo profile-done
