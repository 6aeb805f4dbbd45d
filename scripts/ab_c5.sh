#!/bin/bash
# c5 bench with alternating experiment builds swapped in: ab_c5.sh NAME...
cd "$(dirname "$0")/.."
cp paper_2603_07917_b200/libsagesched.so /tmp/ab_orig.so
for rep in 1 2; do for v in "$@"; do
  cp build_exp/$v/libsagesched.so paper_2603_07917_b200/libsagesched.so
  for c in c5 c3; do
    timeout 300 python bench.py --config $c --no-cpu-baseline 2>/dev/null | python -c "import json,sys; b=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v $c', b['ms_per_step'], b['value'])"
  done
  timeout 300 python bench.py --no-cpu-baseline --no-c4 --no-pure 2>/dev/null | python -c "import json,sys; b=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v c2', b['ms_per_step'], b['e2e']['ms_per_step'])"
done; done
cp /tmp/ab_orig.so paper_2603_07917_b200/libsagesched.so
