#!/bin/bash
# Round-2 measurement session: parity suite, the default bench line, launch list,
# one-frame ncu --set full capture (default sort path) and the summaries.
set -u
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt 2>&1; nproc >> $OUT/smi.txt
if [ "${TESTS:-1}" = "1" ]; then
  timeout 900 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_gpu.log
fi
timeout 600 python bench.py ${BENCH_ARGS:-} > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; tail -3 $OUT/bench.err
python -c "
import json; d=json.loads(open('$OUT/bench.json').read().strip().splitlines()[-1])
print('value', d['value'], 'e2e', d['e2e']['value'] if d.get('e2e') else None, {k: round(v['ms'],4) for k,v in d['stages'].items()})"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file $OUT/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-off --no-inflight --no-cub ${BENCH_ARGS:-} > /dev/null 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on \
  -k "regex:k_raster|k_preprocess|k_upsweep|k_downsweep|k_scan|k_emit|k_ranges|k_tile|k_bucket" \
  -s ${NCU_SKIP:-46} -c ${NCU_COUNT:-23} -o $OUT/prof -f python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-off \
  --no-inflight --no-cub ${BENCH_ARGS:-} > $OUT/ncu_full.log 2>&1
echo "ncu full rc=$?"; tail -2 $OUT/ncu_full.log
