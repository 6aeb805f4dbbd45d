#!/bin/bash
# SHARE-mode bound refresh period (tiles) vs pure top-k time at c2; relinks
# the library with k_topk_sm100_ts.cu rebuilt per setting (default last)
cd "$(dirname "$0")/.."
P=paper_2603_07917_b200
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -I include"
for ev in 1 4 8 16 2; do
  nvcc $F -DSS_SHARE_EVERY=$ev -c -o $P/build_obj/k_topk_sm100_ts.o $P/csrc/k_topk_sm100_ts.cu || exit 1
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o $P/libsagesched.so $P/build_obj/*.o || exit 1
  for th in -1 0.0; do
    echo "every=$ev theta=$th $(timeout 120 python scripts/profile_topk.py --nq 1024 --theta $th --time --reps 10 2>&1 | tail -1)"
  done
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "pure or c2_full or large_batch or edges or round_c1" 2>&1 | tail -1
