#!/bin/bash
# alternate e2e per-call timings of experiment builds: ab_e2e.sh NAME...
cd "$(dirname "$0")/.."
for rep in 1 2 3; do for v in "$@"; do
  timeout 300 python scripts/time_e2e.py --lib build_exp/$v/libsagesched.so --calls ${CALLS:-2000} 2>&1 | tail -1
done; done
