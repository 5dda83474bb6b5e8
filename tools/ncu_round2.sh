#!/usr/bin/env bash
# Round-2 ncu evidence on one B200 (never a bench value): the launch list of the default bench command,
# one --set full capture of the B = 1024 scan, and the B = 1 chain kernels.
set -u
O=gpurun_out/${TAG:-ncu2}; mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $O/launches_bench.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-sweep > $O/ncu_launch_bench.log 2>&1; echo "launch rc=$?" >> $O/summary.txt
#timeout 900 ncu --set full --import-source on --clock-control none -k regex:"ivf_scan_tc" -s 2 -c 1 -o $O/scan_b1024 \
#  python tools/prof_search.py --batch 1024 --searches 3 --no-stages > $O/ncu_scan.log 2>&1; echo "scan rc=$?" >> $O/summary.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"coarse_gemv|coarse_select|plan_small|ivf_scan|merge_rerank|fallback" -s 6 -c 6 -o $O/search_b1 \
  python tools/prof_search.py --batch 1 --searches 3 --no-stages > $O/ncu_b1.log 2>&1; echo "b1 rc=$?" >> $O/summary.txt
cat $O/summary.txt
