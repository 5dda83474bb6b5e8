#!/usr/bin/env bash
# Builds oracle/_ref/ref_harness from the reference's own sources where they lie
# (read-only under /root/reference) — TEST INFRASTRUCTURE, never shipped.
# Only the four core files the harness needs are compiled; the reference's
# CMake build is not used. nlohmann/json (a reference dependency, vendored
# nowhere in /root/reference) comes from the cudnn_frontend copy in the venv.
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
mkdir -p "$here/_ref"
g++ -std=c++20 -O2 -I"$ref/core/include" -I"$json_inc" \
  "$ref/core/src/units.cpp" "$ref/core/src/domain.cpp" "$ref/core/src/memory_planner.cpp" \
  "$ref/core/src/prefetch_timeline.cpp" "$ref/core/src/cost_model.cpp" \
  "$here/ref_harness.cpp" -o "$here/_ref/ref_harness"
echo "built $here/_ref/ref_harness"
