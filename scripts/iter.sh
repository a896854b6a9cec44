#!/bin/bash
# Quick GPU iteration: parity tests + short bench (+ optional env variants).
set -u
mkdir -p gpurun_out
timeout 300 python -m pytest tests -q -m gpu -x 2>&1 | tail -4
for v in "${@:-default}"; do
  if [ "$v" = "default" ]; then env_=""; else env_="$v"; fi
  echo "== $v"
  env $env_ timeout 200 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); st=d['stages']
        print('fps %.1f ms %.3f' % (d['value'], d['ms_per_step']), ' '.join('%s=%.3f' % (k, v['ms']) for k, v in st.items()), 'pairs', d['pairs_per_frame'], 'off', d.get('adagscale_off'))
    else: print(l.rstrip()[:300])
"
done
