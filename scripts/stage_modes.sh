#!/bin/bash
# Per-stage device ms for config 3 AdaGScale on / off and config 1.
for args in "--config 3 --mode adagscale" "--config 3 --mode ellipse" "--config 1 --mode adagscale"; do
  python bench.py $args --steps 50 --warmup 5 --no-cpu --no-e2e --no-off --no-inflight --no-gather 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$args', round(d['value'],1), {k: round(v['ms'],4) for k,v in d['stages'].items()})"
done
