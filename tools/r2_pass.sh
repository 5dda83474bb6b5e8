#!/usr/bin/env bash
# Round-2 GPU pass: smoke, the whole -m gpu suite (no -x, durations), a default bench line.
set -u
O=gpurun_out/${TAG:-r2a}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/gpu.txt 2>&1
timeout 300 python __graft_entry__.py > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/summary.txt
timeout ${PYT:-1500} python -m pytest tests -q -m gpu --durations=25 ${PYTEST_ARGS:-} > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/summary.txt
if [ "${BENCH:-1}" = "1" ]; then
  timeout 900 python bench.py ${BENCH_ARGS:-} > $O/bench.log 2>&1; echo "bench rc=$?" >> $O/summary.txt
fi
cat $O/summary.txt
