#!/bin/bash
# full ncu capture of one launch of kernel regex $1 (run under gpurun); report -> gpurun_out/prof_$2
set -e
CMD="python bench.py --images 2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"$1" -s 3 -c 1 -o gpurun_out/prof_$2 $CMD > gpurun_out/ncu_full_$2.log 2>&1
ncu -i gpurun_out/prof_$2.ncu-rep --page source --csv --print-source sass > gpurun_out/source_$2.csv 2>&1
echo profile-done
