set -x
timeout 600 python -m pytest tests/test_arm_tc_gpu.py tests/test_parity_gpu.py tests/test_arm_decode_gpu.py tests/test_abi.py -x -q 2>&1 | tail -3
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_tcg.json 2> gpurun_out/bench_tcg.err; python -c "
import json; d=json.load(open('gpurun_out/bench_tcg.json')); print(d['value'], d['arm_path'], json.dumps(d['roofline'])); print(json.dumps(d['kernels']))"
