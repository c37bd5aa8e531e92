#!/bin/bash
# The non-headline rows' bench lines (run under gpurun): Table 1, 8K strips,
# training, decoder output stage, ARM decode.   bash tools/bench_rows.sh r02
R=${1:-r02}
: > gpurun_out/bench_table1_$R.jsonl
for c in t300 t545 t1079 t2300; do
  python bench.py --config $c --images 16 --no-cpu-baseline 2>>gpurun_out/bench_rows_$R.err >> gpurun_out/bench_table1_$R.jsonl
done
: > gpurun_out/bench_configs_$R.jsonl
for c in tiny low ref; do
  python bench.py --config $c --images 64 --no-cpu-baseline 2>>gpurun_out/bench_rows_$R.err >> gpurun_out/bench_configs_$R.jsonl
done
python bench.py --config 8k --no-cpu-baseline > gpurun_out/bench_8k_$R.json 2>>gpurun_out/bench_rows_$R.err
python bench.py --train --steps 300 --warmup 10 --no-cpu-baseline > gpurun_out/bench_train_$R.json 2>>gpurun_out/bench_rows_$R.err
python bench.py --train --steps 200 --warmup 10 --images 4 --no-cpu-baseline > gpurun_out/bench_train_multi_$R.json 2>>gpurun_out/bench_rows_$R.err
python bench.py --decode --no-cpu-baseline > gpurun_out/bench_decode_$R.json 2>>gpurun_out/bench_rows_$R.err
python bench.py --arm-decode --no-cpu-baseline > gpurun_out/bench_arm_decode_$R.jsonl 2>>gpurun_out/bench_rows_$R.err
echo rows-done
