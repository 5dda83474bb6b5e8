#!/usr/bin/env bash
# Builds oracle/_ref/ragsim_measured: the reference's own simulator sources, compiled in place from
# /root/reference/proj/core/src (read-only; the reference's CMake build is not used), linked with
# oracle/ragsim_measured.cpp and -Wl,--wrap on retrieval_time / choose_retrieval_batch so the
# retrieval stage can run on measured B200 search times. TEST / EVALUATION INFRASTRUCTURE, never
# shipped. nlohmann/json: the copy bundled in the venv (as in build_ref.sh).
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
ref="${RAGSIM_REF:-/root/reference/proj}"
if [ ! -d "$ref/core/src" ]; then echo "reference not present; skipping _ref build"; exit 0; fi
json_inc="$(python - <<'PY'
import glob, os
c = glob.glob('/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty') + \
    glob.glob('/usr/include')
for d in c:
    if os.path.exists(os.path.join(d, 'nlohmann', 'json.hpp')):
        print(d); break
PY
)"
mkdir -p "$here/_ref/sim_obj"
srcs="units domain memory_planner prefetch_timeline cost_model scheduler simulator workload config_io"
objs=""
for s in $srcs; do
  g++ -std=c++20 -O2 -I"$ref/core/include" -I"$json_inc" -c "$ref/core/src/$s.cpp" -o "$here/_ref/sim_obj/$s.o"
  objs="$objs $here/_ref/sim_obj/$s.o"
done
g++ -std=c++20 -O2 -I"$ref/core/include" -I"$json_inc" -c "$here/ragsim_measured.cpp" -o "$here/_ref/sim_obj/ragsim_measured.o"
g++ -o "$here/_ref/ragsim_measured" "$here/_ref/sim_obj/ragsim_measured.o" $objs \
  -Wl,--wrap=_ZN6ragsim14retrieval_timeEiRKNS_15DatabaseProfileE \
  -Wl,--wrap=_ZN6ragsim22choose_retrieval_batchEii
echo "built $here/_ref/ragsim_measured"
