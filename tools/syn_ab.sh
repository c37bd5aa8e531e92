#!/bin/bash
# Synthesis 1x1 path A/B: the bench's kernel times with CCRD_SYN_PATH=ffma2 and mma.
for path in ffma2 mma; do
  echo -n "syn=$path "
  CCRD_SYN_PATH=$path IMAGES=${IMAGES:-64} bash tools/exp_bench.sh
done
