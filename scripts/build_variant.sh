#!/bin/bash
# build a knob variant of libgtb200.so: scripts/build_variant.sh NAME "-DGT_PR_TILE=4096 ..."
set -e
cd "$(dirname "$0")/.."
name=$1; shift
flags="$*"
mkdir -p build/var_$name
objs=""
for f in paper_1503_07881_b200/csrc/*.cu; do
  o=build/var_$name/$(basename $f .cu).o
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr $flags -c $f -o $o &
  objs="$objs $o"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_1503_07881_b200/libgtb200_$name.so $objs
echo built $name
