#!/usr/bin/env bash
# Round-end evidence pass on one B200: smoke, parity tests, every bench config, the reference
# arm, a batch sweep, the launch list of the default bench command, and one full ncu capture of
# the dominant kernel (scan) at B = 1024 plus the small-batch kernels at B = 1.
set -u
mkdir -p gpurun_out/final
O=gpurun_out/final
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/gpu.txt 2>&1
timeout 300 python __graft_entry__.py > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/summary.txt
timeout 900 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/summary.txt
timeout 900 python bench.py > $O/bench_c2.log 2>&1; echo "bench c2 rc=$?" >> $O/summary.txt
for c in c1 c3 c4 c5; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_$c.log 2>&1; echo "bench $c rc=$?" >> $O/summary.txt
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.log 2>&1; echo "ref rc=$?" >> $O/summary.txt
BATCHES="1 2 4 8 16 32 64 128 256 512 1024" STEPS=30 ./tools/sweep.sh > $O/sweep.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_bench.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-sweep > $O/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"ivf_scan_tc" -s 2 -c 1 -o $O/scan_b1024 \
  python tools/prof_search.py --batch 1024 --searches 3 > $O/ncu_scan.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -s 8 -c 8 -o $O/search_b1 \
  python tools/prof_search.py --batch 1 --searches 3 > $O/ncu_b1.log 2>&1
echo done >> $O/summary.txt
