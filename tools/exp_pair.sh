#!/usr/bin/env bash
# A/B of the paired-CTA wide scan (scan_pair.cu): parity first (bounded), then bench lines
set -u
O=gpurun_out/${TAG:-pair}; mkdir -p $O
timeout 300 python -m pytest -q -x -m gpu tests/test_gpu_parity.py > $O/pytest_parity.log 2>&1; echo "parity rc=$? $(tail -1 $O/pytest_parity.log)" >> $O/res.txt
if grep -q "passed" $O/pytest_parity.log && ! grep -q "failed" $O/pytest_parity.log; then
  timeout 600 python -m pytest -q -x -m gpu tests/ > $O/pytest_all.log 2>&1; echo "all rc=$? $(tail -1 $O/pytest_all.log)" >> $O/res.txt
  for P in 1 0; do
    echo "PAIR=$P $(RD_PAIR=$P BATCHES='128 256 512 1024' STEPS=60 timeout 600 ./tools/sweep.sh | tr '\n' '|')" >> $O/res.txt
  done
  echo "PAIR=1 again $(RD_PAIR=1 BATCHES='1024' STEPS=60 timeout 300 ./tools/sweep.sh)" >> $O/res.txt
fi
cat $O/res.txt
