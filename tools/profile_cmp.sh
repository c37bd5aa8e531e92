#!/bin/bash
set -e
./tools/microbench/mlp_probe > gpurun_out/mlp_plain.log 2>&1
ncu --set full --clock-control none -k regex:"^k" -s 8 -c 1 -o gpurun_out/prof_mlp ./tools/microbench/mlp_probe > gpurun_out/ncu_mlp.log 2>&1
./tools/profile_arm.sh
