#!/bin/bash
# Round-end evidence (run under gpurun): full bench line, ncu launch list of the
# same command, and one `ncu --set full` capture of each hot kernel.
set -e
R=${1:-r01}
python bench.py > gpurun_out/bench_$R.json 2> gpurun_out/bench_$R.err
CMD="python bench.py --images 4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_$R.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$R.csv $CMD > gpurun_out/ncu_launch_$R.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"arm_rate_kernel|synth_kernel" -s 8 -c 2 -o gpurun_out/full_$R $CMD > gpurun_out/ncu_full_$R.log 2>&1
echo done
