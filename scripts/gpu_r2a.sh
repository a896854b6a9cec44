#!/bin/bash
# Round-2 GPU session A: parity suite, sanitizers, ncu captures of K1 and the sort kernels.
set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_gpu.log
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  timeout 600 $CS --tool $tool --print-limit 50 python scripts/sanitize_workload.py > $OUT/sanitizer_$tool.log 2>&1
  echo "$tool rc=$?"; tail -2 $OUT/sanitizer_$tool.log
done
AGSX_SORT=bucket timeout 600 $CS --tool memcheck --print-limit 50 python scripts/sanitize_workload.py > $OUT/sanitizer_memcheck_bucket.log 2>&1
echo "memcheck bucket rc=$?"; tail -2 $OUT/sanitizer_memcheck_bucket.log
AGSX_SORT=bucket timeout 600 $CS --tool racecheck --print-limit 50 python scripts/sanitize_workload.py > $OUT/sanitizer_racecheck_bucket.log 2>&1
echo "racecheck bucket rc=$?"; tail -2 $OUT/sanitizer_racecheck_bucket.log
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_preprocess|k_upsweep|k_downsweep|k_emit|k_scan" \
  -s 40 -c 16 -o $OUT/prof_k1sort -f python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-off --no-inflight --no-cub > $OUT/ncu_k1.log 2>&1
echo "ncu k1 rc=$?"
AGSX_SORT=bucket timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_preprocess|k_tile_scan|k_bucket_scatter|k_tile_sort" \
  -s 20 -c 4 -o $OUT/prof_bucket -f python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-off --no-inflight --no-cub > $OUT/ncu_bucket.log 2>&1
echo "ncu bucket rc=$?"
