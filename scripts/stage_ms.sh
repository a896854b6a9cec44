#!/bin/bash
# Per-stage device ms of a short config-3 bench for each env variant given.
for v in "$@"; do
  if [ "$v" = "default" ]; then env_=""; else env_="$v"; fi
  env $env_ python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e --no-off > gpurun_out/sm.json 2> gpurun_out/sm.err
  python - "$v" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/sm.json").read().strip().splitlines()[-1])
print(sys.argv[1], round(d["value"], 1), {k: round(v["ms"], 4) for k, v in d["stages"].items()})
PY
done
