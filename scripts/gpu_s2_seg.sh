#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
T=${1:-s2seg}
for V in "" seg3 seg2; do
  GT_LIB_VARIANT=$V timeout 300 python scripts/prof_build.py c4 2 > gpurun_out/${T}_c4_${V:-base}.log 2>&1
done
echo done
