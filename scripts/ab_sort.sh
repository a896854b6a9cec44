#!/bin/bash
# A/B of the sort paths on one box: parity subset, then bench lines per variant.
#   VARIANTS="bucket depth" bash scripts/ab_sort.sh
set -u
OUT=gpurun_out
mkdir -p $OUT
if [ "${TESTS:-1}" = "1" ]; then
  timeout 600 python -m pytest tests -m gpu -x -q -k "${TEST_K:-small or config1 or config3}" > $OUT/pytest_gpu.log 2>&1
  echo "pytest rc=$?"; tail -2 $OUT/pytest_gpu.log
fi
summ() {
  python - "$1" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d["value"], 1), {k: round(v["ms"], 4) for k, v in d["stages"].items()},
      "off", round((d.get("adagscale_off") or {}).get("fps_per_gpu", 0), 1))
PY
}
for v in ${VARIANTS:-bucket depth}; do
  case $v in
    depth) AGSX_SORT=depth timeout 300 python bench.py --steps 20 --no-cpu --no-e2e --no-inflight > $OUT/b_$v.json 2> $OUT/b_$v.err ;;
    bucket) AGSX_SORT=bucket timeout 300 python bench.py --steps 20 --no-cpu --no-e2e --no-inflight > $OUT/b_$v.json 2> $OUT/b_$v.err ;;
    *) timeout 300 python bench.py --steps 20 --no-cpu --no-e2e --no-inflight > $OUT/b_$v.json 2> $OUT/b_$v.err ;;
  esac
  summ $OUT/b_$v.json || tail -3 $OUT/b_$v.err
done
if [ "${NCU:-0}" = "1" ]; then
  timeout 400 ncu --set full --clock-control none --import-source on -k "regex:${NCU_KERNELS:-k_tile_sort|k_bucket_scatter|k_tile_scan|k_preprocess}" \
    -s ${NCU_SKIP:-12} -c ${NCU_COUNT:-4} -o $OUT/prof -f python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-off --no-inflight > $OUT/ncu_full.log 2>&1
  echo "ncu rc=$?"
fi
