#!/bin/bash
# Bench experiment variants of libccrd (tools/libccrd_*.so) back to back; prints kernel times.
for lib in "" $@; do
  if [ -n "$lib" ]; then export CCRD_LIB=$PWD/$lib; else unset CCRD_LIB; fi
  python bench.py --images ${IMAGES:-16} --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>gpurun_out/exp_err_$(basename "${lib:-main}").log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']
a=[v for n,v in k.items() if n.startswith('arm_')][0]
print('${lib:-main}', round(d['value']/1e9,3), 'Gpx/s', 'arm', round(a['avg_launch_ms']*1e3,1), 'us', round(a['frac'],3), 'syn', round(k['synth_kernel']['avg_launch_ms']*1e3,1), 'us', round(k['synth_kernel']['frac'],3), 'pyr/step', round(k.get('pyramid_kernel',{}).get('ms_total',0)*1e3/d['steps'],1), 'us')"
done
