#!/usr/bin/env bash
# Latency pass: GPU parity tests, batch sweep, per-kernel launch lists at small batches.
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" > gpurun_out/summary.txt
tail -3 gpurun_out/pytest_gpu.log >> gpurun_out/summary.txt
BATCHES="${BATCHES:-1 8 32 64 128 1024}" STEPS=30 ./tools/sweep.sh > gpurun_out/sweep.txt 2>&1
for v in ${AB_VARIANTS:-}; do echo "== $v" >> gpurun_out/sweep.txt; env $v BATCHES="${AB_BATCHES:-256 1024}" STEPS=30 ./tools/sweep.sh >> gpurun_out/sweep.txt 2>&1; done
for B in ${LAUNCH_BATCHES:-1 8}; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_b$B.csv \
    python tools/prof_search.py --batch $B --searches 3 > gpurun_out/prof_b$B.log 2>&1
done
