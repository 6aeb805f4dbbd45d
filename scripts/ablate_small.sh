#!/bin/bash
# small-batch (streaming scan) timing of the stage-1 kernel for SS_TC_DEBUG values
cd "$(dirname "$0")/.."
nq=${NQ:-8}
for d in "$@"; do
  echo "nq=$nq dbg=$d $(SS_TC_DEBUG=$d timeout 90 python scripts/profile_topk.py --nq $nq --time --reps 50 2>&1 | tail -1)"
done
