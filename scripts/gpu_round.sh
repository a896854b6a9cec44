#!/bin/bash
# One GPU session: tests, bench, ncu launch list + full captures. Outputs in gpurun_out/.
set -u
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt 2>&1; nproc >> $OUT/smi.txt
if [ "${TESTS:-1}" = "1" ]; then
  timeout ${TEST_TIMEOUT:-420} python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; rc=$?; echo "pytest rc=$rc"
  if [ $rc -eq 124 ]; then echo "tests timed out: stopping"; tail -20 $OUT/pytest_gpu.log; exit 1; fi
  tail -5 $OUT/pytest_gpu.log
  if grep -q "rc=124" <<< "$(tail -1 $OUT/pytest_gpu.log)"; then :; fi
fi
if [ "${BENCH:-1}" = "1" ]; then
  timeout ${BENCH_TIMEOUT:-240} python bench.py ${BENCH_ARGS:-} > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
  tail -c 3000 $OUT/bench.json; tail -3 $OUT/bench.err
fi
if [ "${NCU:-1}" = "1" ]; then
  timeout 240 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-off --no-inflight > /dev/null 2>&1; echo "ncu list rc=$?"
  timeout ${NCU_TIMEOUT:-420} ncu --set full --clock-control none --import-source on -k "regex:${NCU_KERNELS:-k_raster|k_preprocess|k_upsweep|k_downsweep|k_scan|k_emit|k_ranges}" \
    -s ${NCU_SKIP:-23} -c ${NCU_COUNT:-23} -o $OUT/prof -f python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-off --no-inflight > $OUT/ncu_full.log 2>&1
  echo "ncu full rc=$?"; tail -3 $OUT/ncu_full.log
fi
