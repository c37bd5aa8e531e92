#!/bin/bash
# e2e (host-buffer path) A/B: the bench's e2e value under environment variants.
#   bash tools/exp_e2e.sh "CCRD_WIDEN_STREAM=0" "CCRD_WIDEN_STREAM=1"
for v in "$@"; do
  env $v python bench.py --steps 3 --warmup 3 --e2e-steps 5 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', 'device', round(d['value']/1e9,3), 'e2e', round(d['e2e']['value']/1e9,3), 'Gpx/s')"
done
