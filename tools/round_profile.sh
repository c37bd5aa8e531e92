#!/bin/bash
# Round-end evidence (run under gpurun): full bench line, ncu launch list of the
# same command, and one `ncu --set full` capture of each hot kernel.
#   bash tools/round_profile.sh r01 [--full-only]
set -e
R=${1:-r02}
CMD="python bench.py --images 4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
if [ "$2" != "--full-only" ]; then
  python bench.py > gpurun_out/bench_$R.json 2> gpurun_out/bench_$R.err
  $CMD > gpurun_out/plain_$R.log 2>&1
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$R.csv $CMD > gpurun_out/ncu_launch_$R.log 2>&1
fi
for k in arm_tcp_kernel synth_kernel pyramid_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:"$k" -s 2 -c 1 -o gpurun_out/full_${R}_$k $CMD > gpurun_out/ncu_full_${R}_$k.log 2>&1
done
echo done
