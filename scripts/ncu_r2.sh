#!/bin/bash
# ncu --set full captures of the round-2 kernels (one launch each) -> gpurun_out/
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on"
$NCU -k regex:k_refresh -s 1 -c 1 -o gpurun_out/r2_refresh -f python bench.py --config c3 --steps 2 --warmup 3 > gpurun_out/ncu_refresh.log 2>&1
$NCU -k regex:k_topk_ts -s 1 -c 1 -o gpurun_out/r2_ts -f python scripts/profile_topk.py --nq 1024 --reps 2 > gpurun_out/ncu_ts.log 2>&1
$NCU -k regex:k_topk_tc -s 1 -c 1 -o gpurun_out/r2_scan8 -f python scripts/profile_topk.py --nq 8 --reps 2 > gpurun_out/ncu_scan8.log 2>&1
$NCU -k regex:k_topk_ts -s 1 -c 1 -o gpurun_out/r2_ts_pure -f python scripts/profile_topk.py --nq 1024 --theta -1 --reps 2 > gpurun_out/ncu_ts_pure.log 2>&1
ls -la gpurun_out/*.ncu-rep
