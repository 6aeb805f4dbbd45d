#!/bin/bash
# Ablation of the top-k kernel (SS_TC_DEBUG bits) at c2 and c4 shapes.
# bit 1: no heap path; 2: no MMA; 4: drain only (no epilogue math); 16: no drain
cd "$(dirname "$0")/.."
for ts in 1 0; do
  for d in 0 1 4 16 2 6 18; do
    echo "TS=$ts dbg=$d $(SS_TC_TS=$ts SS_TC_DEBUG=$d python scripts/profile_topk.py --nq 1024 --time --reps 20 2>&1 | tail -1)"
  done
done
for d in 0 1 4 16 2; do
  echo "c4-shape dbg=$d $(SS_TC_DEBUG=$d python scripts/profile_topk.py --nq 8192 --rows 4194304 --time --reps 3 2>&1 | tail -1)"
done
echo "theta=-1 $(python scripts/profile_topk.py --nq 1024 --theta -1 --time --reps 10 2>&1 | tail -1)"
for nq in 8 64 128 256 512; do
  echo "nq=$nq $(python scripts/profile_topk.py --nq $nq --time --reps 20 2>&1 | tail -1)"
done
