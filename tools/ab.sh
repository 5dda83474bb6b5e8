#!/usr/bin/env bash
# A/B of engine builds on one box: VARIANTS="name=path[:ENV=V] ..." (path "-" = the in-tree build),
# BATCHES, REPS; prints one line per (rep, batch, variant)
for rep in $(seq ${REPS:-2}); do
  for B in ${BATCHES:-64 1024}; do
    for v in ${VARIANTS:-cur=-}; do
      name=${v%%=*}; rest=${v#*=}; path=${rest%%:*}; envs=""
      [[ "$rest" == *:* ]] && envs=${rest#*:}
      if [ "$path" = "-" ]; then unset RD_ENGINE_PATH; else export RD_ENGINE_PATH=$PWD/$path; fi
      env ${envs//,/ } timeout 300 python bench.py --steps ${STEPS:-40} --warmup 3 --no-cpu-baseline --no-sweep --batch $B 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('B=%5d %-10s q/s=%9.0f e2e=%9.0f scan_ms=%.3f mhz=%s %s' % ($B, '$name', d['value'], d['e2e']['value'], r['avg_launch_ms'], d['clocks']['sm_mhz'], d['clocks']['reasons']))"
    done
  done
done
unset RD_ENGINE_PATH
