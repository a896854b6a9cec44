#!/bin/bash
# Round-2 evidence session: parity suite (both sort paths), sanitizers (fixed
# racecheck), the default bench line, launch list, one-frame ncu --set full, and a
# memcheck of one full config-3 frame.
set -u
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt 2>&1; nproc >> $OUT/smi.txt
timeout 900 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 $OUT/pytest_gpu.log
AGSX_SORT=bucket timeout 900 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu_bucket.log 2>&1; echo "pytest bucket rc=$?"; tail -1 $OUT/pytest_gpu_bucket.log
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  timeout 600 $CS --tool $tool --print-limit 50 python scripts/sanitize_workload.py > $OUT/sanitizer_$tool.log 2>&1
  echo "$tool rc=$?"; tail -1 $OUT/sanitizer_$tool.log
done
for tool in memcheck racecheck; do
  AGSX_SORT=bucket timeout 600 $CS --tool $tool --print-limit 50 python scripts/sanitize_workload.py > $OUT/sanitizer_${tool}_bucket.log 2>&1
  echo "$tool bucket rc=$?"; tail -1 $OUT/sanitizer_${tool}_bucket.log
done
timeout 900 $CS --tool memcheck --print-limit 20 python scripts/memcheck_c3.py > $OUT/sanitizer_memcheck_config3.log 2>&1
echo "memcheck config3 rc=$?"; tail -1 $OUT/sanitizer_memcheck_config3.log
BENCH_ARGS="${BENCH_ARGS:-}" TESTS=0 bash scripts/gpu_r2b.sh
