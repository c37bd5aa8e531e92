#!/bin/bash
# End-to-end (host-buffer) A/B of the in-tree library against a variant build
# of the same ABI (run under gpurun):  bash tools/e2e_ab.sh tools/libccrd_X.so
VAR=${1:?usage: tools/e2e_ab.sh <variant libccrd .so>}
for lib in "" "$VAR" "" "$VAR"; do
  if [ -n "$lib" ]; then export CCRD_LIB=$PWD/$lib; else unset CCRD_LIB; fi
  for c in t300 ref; do
    python bench.py --config $c --images 16 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('${lib:-main}', '$c', '%.4e'%d['value'], 'e2e %.4e'%d['e2e']['value'])"
  done
done
