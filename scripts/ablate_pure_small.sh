#!/bin/bash
cd "$(dirname "$0")/.."
for d in 0 1; do
  echo "nq=8 theta=-1 dbg=$d $(SS_TC_DEBUG=$d timeout 90 python scripts/profile_topk.py --nq 8 --theta -1 --time --reps 20 2>&1 | tail -1)"
done
echo "nq=8 theta=-1 scan $(timeout 90 python scripts/profile_topk.py --nq 8 --theta -1 --algo scan --time --reps 20 2>&1 | tail -1)"
echo "nq=8 theta=0.8 scan $(timeout 90 python scripts/profile_topk.py --nq 8 --theta 0.8 --algo scan --time --reps 20 2>&1 | tail -1)"
