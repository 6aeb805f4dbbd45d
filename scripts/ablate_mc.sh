#!/bin/bash
# TS kernel tile shapes with and without 2-CTA multicast clusters at c2
# (SS_TC_MC; SS_TC_TSN=512: 256 x 2 accumulators, A in shared memory)
cd "$(dirname "$0")/.."
for tsn in 208 512; do
  for mc in 0 1; do
    for d in 0 16 64; do
      echo "TSN=$tsn MC=$mc dbg=$d $(SS_TC_TSN=$tsn SS_TC_MC=$mc SS_TC_DEBUG=$d timeout 90 python scripts/profile_topk.py --nq 1024 --time --reps 20 2>&1 | tail -1)"
    done
  done
done
