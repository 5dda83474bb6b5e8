#!/usr/bin/env bash
# Every bench config on one GPU (C1, C2 default line, C3, C4 one stripe of 8, C5, C2 under an 8B reservation)
set -u
O=gpurun_out/${TAG:-r2cfg}
mkdir -p $O
for c in ${CONFIGS_LIST:-c2 c1 c3 c4 c5 c2r8b}; do
  extra=""; [ "$c" != c2 ] && extra="--steps 10 --warmup 3 --no-cpu-baseline"
  timeout 900 python bench.py --config $c $extra > $O/bench_$c.log 2>&1; echo "bench $c rc=$?" >> $O/summary.txt
done
cat $O/summary.txt
