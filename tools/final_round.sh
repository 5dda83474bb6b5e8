#!/usr/bin/env bash
# Round-end evidence pass on one B200: smoke, the GPU test suite, every bench config, the reference
# arm, a batch sweep, the launch list of the default bench command, and full ncu captures of the
# B = 1024 scan and the B = 1 chain. Outputs under gpurun_out/${TAG:-final2}.
set -u
O=gpurun_out/${TAG:-final2}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/gpu.txt 2>&1
timeout 300 python __graft_entry__.py > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/summary.txt
timeout 900 python -m pytest tests -q -m gpu --durations=15 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/summary.txt
timeout 900 python bench.py > $O/bench_c2.log 2>&1; echo "bench c2 rc=$?" >> $O/summary.txt
for c in c1 c3 c4 c5 c2r8b; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_$c.log 2>&1; echo "bench $c rc=$?" >> $O/summary.txt
done
timeout 900 python bench.py --impl reference --steps 20 --warmup 3 > $O/bench_ref.log 2>&1; echo "ref rc=$?" >> $O/summary.txt
BATCHES="1 2 4 8 16 32 64 128 256 512 1024" STEPS=40 ./tools/sweep.sh > $O/sweep.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $O/launches_bench.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-sweep > $O/ncu_launch_bench.log 2>&1; echo "launch rc=$?" >> $O/summary.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"ivf_scan_tc" -s 2 -c 1 -o $O/scan_b1024 \
  python tools/prof_search.py --batch 1024 --searches 3 --no-stages > $O/ncu_scan.log 2>&1; echo "ncu scan rc=$?" >> $O/summary.txt
timeout 900 ncu --set full --import-source on --clock-control none \
  -k regex:"coarse_gemv|coarse_select|plan_small|ivf_scan|merge_rerank|fallback" -s 5 -c 5 -o $O/search_b1 \
  python tools/prof_search.py --batch 1 --searches 3 --no-stages > $O/ncu_b1.log 2>&1; echo "ncu b1 rc=$?" >> $O/summary.txt
echo done >> $O/summary.txt
cat $O/summary.txt
