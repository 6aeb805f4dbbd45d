#!/bin/bash
# onesweep rank: look-back window vs the c3 round (see exp_rank_items.sh)
cd "$(dirname "$0")/.."
P=paper_2603_07917_b200
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -I include"
for lb in 16 32 8; do
  nvcc $F -DSS_OS_LB=$lb -c -o $P/build_obj/k_rank.o $P/csrc/k_rank.cu || exit 1
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o $P/libsagesched.so $P/build_obj/*.o || exit 1
  for r in 1 2; do
    echo "lb=$lb $(timeout 300 python bench.py --config c3 2>/dev/null | tail -1 | python -c 'import json,sys;d=json.loads(sys.stdin.read());print(d["ms_per_step"])')"
  done
  timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "rank or c3" 2>&1 | tail -1
done
