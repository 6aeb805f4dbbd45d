#!/bin/bash
# warp-cooperative exact path (SS_TC_DEBUG=512) vs default at c2: parity + time
cd "$(dirname "$0")/.."
echo "parity: $(SS_TC_DEBUG=512 timeout 300 python scripts/check_topk_variant.py 30000 1000 2>&1 | tail -1)"
echo "parity: $(SS_TC_DEBUG=512 timeout 300 python scripts/check_topk_variant.py 100003 600 2>&1 | tail -1)"
for r in 1 2; do
  for d in 0 512; do
    echo "dbg=$d $(SS_TC_DEBUG=$d timeout 90 python scripts/profile_topk.py --nq 1024 --time --reps 20 2>&1 | tail -1)"
  done
done
