#!/usr/bin/env bash
# Round-2 bench pass: default bench line (C2) and the reference arm, on one B200.
set -u
O=gpurun_out/${TAG:-r2bench}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/gpu.txt 2>&1
nproc > $O/nproc.txt; grep -m1 "model name" /proc/cpuinfo >> $O/nproc.txt
timeout 900 python bench.py ${BENCH_ARGS:-} > $O/bench.log 2>&1; echo "bench rc=$?" >> $O/summary.txt
timeout 900 python bench.py --impl reference ${REF_ARGS:---steps 20 --warmup 3} > $O/bench_ref.log 2>&1; echo "ref rc=$?" >> $O/summary.txt
cat $O/summary.txt
