#!/bin/bash
# quick top-k kernel timing at c2 (nq=1024) for a list of SS_TC_DEBUG values
cd "$(dirname "$0")/.."
for d in "$@"; do
  echo "dbg=$d $(SS_TC_DEBUG=$d timeout 90 python scripts/profile_topk.py --nq 1024 --time --reps 20 2>&1 | tail -1)"
done
