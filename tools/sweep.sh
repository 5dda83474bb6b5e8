#!/usr/bin/env bash
# batch sweep of the bench (config c2), one JSON line per run
for B in ${BATCHES:-1 8 32 64 128 256 512 1024}; do
  timeout 300 python bench.py --steps ${STEPS:-30} --warmup 3 --batch $B --no-cpu-baseline --no-sweep ${EXTRA:-} 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('B=%5d q/s=%10.0f e2e=%10.0f ms=%7.3f scan_ms=%6.3f scanGBs=%6.0f frac=%.3f coarse_ms=%.3f sm_mhz=%s %s' % (d['config']['global_batch'], d['value'], d['e2e']['value'], d['ms_per_step'], r['avg_launch_ms'], r['achieved'], r['frac'], d['step_breakdown_ms']['coarse_ms'], d['clocks']['sm_mhz'], d['clocks']['reasons']))"
done
