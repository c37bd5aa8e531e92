#!/bin/bash
# A/B of the synthesis staging paths on the headline workload (run under gpurun):
# per-tile LDG kernel (ffma2) vs TMA-staged persistent CTAs (tma, 1 / 2 CTAs per SM).
CMD="python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline"
VARS=${AB_VARIANTS:-"ffma2:2 tma:2 tma:1 ffma2:2 tma:2"}
for v in $VARS; do
  v=${v/:/ }
  set -- $v
  echo "== path=$1 pctas=$2"
  CCRD_SYN_PATH=$1 CCRD_SYN_PCTAS=$2 $CMD 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
k=d['kernels']
print('value %.4e  synth %.1f us  arm %.1f us  frac %.3f' % (d['value'], k['synth_kernel']['avg_launch_ms']*1e3, k.get('arm_tcp_kernel', k.get('arm_tcg_kernel'))['avg_launch_ms']*1e3, d['roofline']['frac']))"
done
