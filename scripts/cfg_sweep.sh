#!/bin/bash
# Device FPS of every BASELINE config (and AdaGScale off) with the current build:
#   bash scripts/cfg_sweep.sh > gpurun_out/sweep.txt
set -u
for c in 1 2 3 4 5; do
  for m in adagscale ellipse $([ $c = 2 ] && echo aabb_fixed3); do
    echo -n "config $c $m: "
    timeout 300 python bench.py --config $c --mode $m --steps 20 --warmup 3 --no-cpu --no-e2e --no-off --no-inflight --no-cub 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); st=d['stages']
        print('fps %.1f' % d['value'], ' '.join('%s=%.4f' % (k, v['ms']) for k, v in st.items()), 'pairs', d['pairs_per_frame'])"
  done
done
