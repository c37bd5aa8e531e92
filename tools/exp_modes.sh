#!/bin/bash
# bench variants (tools/libccrd_*.so or main) in concurrent and serial stream modes
for lib in "" $@; do
  for mode in conc serial; do
    if [ -n "$lib" ]; then export CCRD_LIB=$PWD/$lib; else unset CCRD_LIB; fi
    if [ "$mode" = serial ]; then export CCRD_SERIAL=1; else unset CCRD_SERIAL; fi
    python bench.py --images ${IMAGES:-32} --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']
print('${lib:-main}', '$mode', round(d['value']/1e9,3), 'Gpx/s', 'arm', round(k['arm_rate_kernel']['avg_ms']*1e3,1), 'syn', round(k['synth_kernel']['avg_ms']*1e3,1), 'us (serial pass)')"
  done
done
unset CCRD_SERIAL CCRD_LIB
