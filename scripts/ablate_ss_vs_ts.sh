#!/bin/bash
# SS (A in smem, N=256 x 2 accumulators) vs TS (A in TMEM, N=208 x 2) at c2:
# full kernel, no drain (MMA + TMA floor), MMA issue alone
cd "$(dirname "$0")/.."
for ts in 0 1; do
  for d in 0 16 64 72; do
    echo "TS=$ts dbg=$d $(SS_TC_TS=$ts SS_TC_DEBUG=$d timeout 90 python scripts/profile_topk.py --nq 1024 --time --reps 20 2>&1 | tail -1)"
  done
done
