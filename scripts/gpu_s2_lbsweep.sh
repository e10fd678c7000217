#!/bin/bash
# look-back window / occupancy variants of the sort kernels (C4 build timings)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
T=${1:-s2lb}
for V in "" lb2 lb8 lb16 b5; do
  for P in 0 1; do
    GT_LIB_VARIANT=$V GT_SORT_PIPE=$P timeout 300 python scripts/prof_build.py c4 2 > gpurun_out/${T}_${V:-base}_k$P.log 2>&1
  done
done
echo done
