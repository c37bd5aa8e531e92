#!/bin/bash
# ncu launch list + full capture of the two hot kernels (run under gpurun).
set -e
CMD="python bench.py --images 4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"arm_rate_kernel|synth_kernel" -s 8 -c 2 -o gpurun_out/prof_r01 $CMD > gpurun_out/ncu_full.log 2>&1
echo profile-done
