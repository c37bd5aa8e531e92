for pp in 0 1; do CCRD_ARM_TC_PP=$pp IMAGES=16 bash tools/exp_bench.sh; done
CCRD_ARM_TC_PP=1 IMAGES=16 bash tools/exp_bench.sh tools/libccrd_pp80.so | tail -1
CCRD_ARM_TC_PP=1 IMAGES=64 bash tools/exp_bench.sh
