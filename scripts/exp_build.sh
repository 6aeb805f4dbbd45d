#!/bin/bash
# Build experiment variants of libsagesched: exp_build.sh NAME "-DFLAG=V ..." -> build_exp/NAME/libsagesched.so
cd "$(dirname "$0")/.."
name=$1; shift
flags="$*"
out=build_exp/$name; mkdir -p $out
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -I include"
objs=""
for f in paper_2603_07917_b200/csrc/*.cu; do
  o=$out/$(basename $f .cu).o
  nvcc $F $flags -c -o $o $f &
  objs="$objs $o"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o $out/libsagesched.so $objs && echo "built $out"
