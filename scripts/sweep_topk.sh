#!/bin/bash
# stage-1 kernel time across theta, k and batch size (1M-row bank)
cd "$(dirname "$0")/.."
for th in 0.9 0.8 0.6 0.3 0.0 -1; do
  echo "theta=$th k=64 $(timeout 120 python scripts/profile_topk.py --nq 1024 --theta $th --time --reps 10 2>&1 | tail -1)"
done
for k in 16 32 128; do
  echo "theta=0.8 k=$k $(timeout 120 python scripts/profile_topk.py --nq 1024 --k $k --time --reps 10 2>&1 | tail -1)"
done
for nq in 1 8 64 128 256 512 2048 4096 8192; do
  echo "theta=0.8 nq=$nq $(timeout 120 python scripts/profile_topk.py --nq $nq --time --reps 10 2>&1 | tail -1)"
done
