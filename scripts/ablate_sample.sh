#!/bin/bash
# pure top-k warm start (SS_TC_SAMPLE) at c2, theta = -1 and 0
cd "$(dirname "$0")/.."
for th in -1 0.0; do
  for smp in 1 0; do
    echo "theta=$th sample=$smp $(SS_TC_SAMPLE=$smp timeout 120 python scripts/profile_topk.py --nq 1024 --theta $th --time --reps 10 2>&1 | tail -1)"
  done
done
echo "theta=0.8 $(timeout 120 python scripts/profile_topk.py --nq 1024 --time --reps 10 2>&1 | tail -1)"
