#!/bin/bash
# A/B of the synthesis variants on the headline workload (run under gpurun):
#   AB_VARIANTS="ffma2 tma tma:clu" bash tools/syn_tma_ab.sh
# ffma2 = per-tile kernel with clamped LDG staging, tma = TMA-staged interior
# tiles (the default), tma:clu = + vertical tile pairs in 2-CTA clusters.
CMD="python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline"
VARS=${AB_VARIANTS:-"ffma2 tma ffma2 tma"}
for v in $VARS; do
  path=${v%%:*}
  clu=0; [ "$v" != "${v%:clu}" ] && clu=1
  echo "== path=$path clusters=$clu"
  CCRD_SYN_PATH=$path CCRD_SYN_CLU=$clu $CMD 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
k=d['kernels']
a=k.get('arm_tcp_kernel', k.get('arm_tcg_kernel'))
print('value %.4e  synth %.1f us  arm %.1f us  frac %.3f' % (d['value'], k['synth_kernel']['avg_launch_ms']*1e3, a['avg_launch_ms']*1e3, d['roofline']['frac']))"
done
