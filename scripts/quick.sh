#!/bin/bash
# Quick GPU iteration: a parity subset, then short bench lines (default and env variants).
#   TEST_K="small or config3" bash scripts/quick.sh "" "AGSX_SORT=bucket"
set -u
mkdir -p gpurun_out
if [ -n "${TEST_K:-small or config1 or config3}" ]; then
  timeout 600 python -m pytest tests -q -m gpu -x -k "${TEST_K:-small or config1 or config3}" 2>&1 | tail -3
fi
for v in "$@"; do
  echo "== ${v:-default}"
  env $v timeout 200 python bench.py --steps 50 --warmup 5 --no-cpu --no-e2e --no-inflight --no-cub ${BENCH_ARGS:-} 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); st=d['stages']
        print('fps %.1f ms %.4f' % (d['value'], d['ms_per_step']), ' '.join('%s=%.4f' % (k, v['ms']) for k, v in st.items()), 'pairs', d['pairs_per_frame'], 'off', (d.get('adagscale_off') or {}).get('fps_per_gpu'))
    elif 'Error' in l or 'error' in l: print(l.rstrip()[:300])
"
done
