set -x
timeout 900 python -m pytest tests/test_arm_tc_gpu.py tests/test_parity_gpu.py tests/test_arm_decode_gpu.py -x -q 2>&1 | tail -3
IMAGES=64 bash tools/exp_bench.sh
