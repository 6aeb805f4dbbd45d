#!/bin/bash
# time the stage-1 kernel for each experiment build: exp_run.sh NAME... (env NQ, THETA, ROWS, REPS)
cd "$(dirname "$0")/.."
for name in "$@"; do
  for th in ${THETAS:-0.8 -1}; do
    echo "$name theta=$th $(timeout 120 python scripts/profile_topk.py --lib build_exp/$name/libsagesched.so --nq ${NQ:-1024} --rows ${ROWS:-1048576} --theta $th --time --reps ${REPS:-30} 2>&1 | tail -1)"
  done
done
