#!/usr/bin/env bash
# Small-batch chain evidence on one B200: per-kernel globaltimer timeline (RD_DEBUG_CHAIN) of a few
# searches at B = 1 and 8, the bench sweep at B <= 64, and the launch list at B = 1 / 8.
set -u
O=gpurun_out/${TAG:-small}
mkdir -p $O
for B in 1 8; do
  RD_DEBUG_CHAIN=1 timeout 300 python tools/prof_search.py --batch $B --searches 6 --no-stages > $O/chain_b$B.log 2>&1
done
BATCHES="1 2 4 8 16 32 64" STEPS=50 ./tools/sweep.sh > $O/sweep.txt 2>&1
for B in 1 8; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_b$B.csv \
    python tools/prof_search.py --batch $B --searches 6 --no-stages > /dev/null 2>&1
done
cat $O/sweep.txt
