#!/bin/bash
# TS kernel bank-stage ring depth (SS_TS_STAGES) at c2, k = 64 and k = 16
cd "$(dirname "$0")/.."
for k in 64 16; do
  for st in 3 4 5 6 8; do
    echo "k=$k stages<=$st $(SS_TS_STAGES=$st timeout 120 python scripts/profile_topk.py --nq 1024 --k $k --time --reps 10 2>&1 | tail -1)"
  done
done
