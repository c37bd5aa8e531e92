#!/bin/bash
# full ncu capture of one training-step kernel (regex $1) -> gpurun_out/prof_train_$2
set -e
CMD="python bench.py --train --steps 1 --warmup 2"
ncu --set full --clock-control none --import-source on -k regex:"$1" -s 1 -c 1 -o gpurun_out/prof_train_$2 $CMD > gpurun_out/ncu_train_$2.log 2>&1
ncu -i gpurun_out/prof_train_$2.ncu-rep --page source --csv --print-source sass > gpurun_out/source_train_$2.csv 2>&1
echo done
