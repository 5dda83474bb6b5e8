#!/usr/bin/env bash
# A/B on one box: alternate RD_DEBUG_SKIP variants, B in $BATCHES
for rep in 1 2; do for m in ${VARIANTS:-0 8}; do
  echo -n "skip=$m "; RD_DEBUG_SKIP=$m BATCHES="${BATCHES:-1024}" STEPS=${STEPS:-40} ./tools/sweep.sh 2>&1
done; done
