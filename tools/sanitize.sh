#!/usr/bin/env bash
# compute-sanitizer over the smoke search and the GPU test suite (round-2 code paths: split3 store,
# fused B = 1 plan, deferred flush, staged merge decode, pair scan). Outputs gpurun_out/${TAG:-san}.
set -u
O=gpurun_out/${TAG:-san}; mkdir -p $O
for tool in racecheck synccheck initcheck; do
  echo "== compute-sanitizer --tool $tool python __graft_entry__.py (smoke)" >> $O/sanitizer.txt
  timeout 900 compute-sanitizer --tool $tool python __graft_entry__.py 2>&1 | grep -E "smoke ok|SUMMARY|Error|error" | head -5 >> $O/sanitizer.txt
done
echo "== compute-sanitizer --tool memcheck python -m pytest tests -m gpu -q (RD_PAIR off and on)" >> $O/sanitizer.txt
timeout 2400 compute-sanitizer --tool memcheck python -m pytest tests -m gpu -q -p no:cacheprovider > $O/memcheck.log 2>&1
grep -E "passed|failed|SUMMARY" $O/memcheck.log | tail -3 >> $O/sanitizer.txt
echo "== compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -m gpu" >> $O/sanitizer.txt
timeout 1500 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -m gpu -q \
  -p no:cacheprovider -k "not read_bandwidth" > $O/racecheck.log 2>&1
grep -E "passed|failed|RACECHECK SUMMARY" $O/racecheck.log | tail -2 >> $O/sanitizer.txt
cat $O/sanitizer.txt
