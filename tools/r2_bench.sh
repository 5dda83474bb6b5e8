#!/usr/bin/env bash
# Round-2 bench pass: default C2 line, the group path (2 stripes on one GPU), the reference arm.
set -u
O=gpurun_out/${TAG:-r2b}
mkdir -p $O
timeout 900 python bench.py ${BENCH_ARGS:-} > $O/bench_c2.log 2>&1; echo "bench c2 rc=$?" >> $O/summary.txt
RD_BENCH_DEVICES=0,0 timeout 600 python bench.py --gpus 2 --config c1 --steps 10 > $O/bench_c1_group2.log 2>&1; echo "group rc=$?" >> $O/summary.txt
timeout 900 python bench.py --impl reference --steps 20 --warmup 3 > $O/bench_ref.log 2>&1; echo "ref rc=$?" >> $O/summary.txt
cat $O/summary.txt
