#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
T=${1:-s2tch}
for V in "" ch128 ch512 ch1024; do
  GT_LIB_VARIANT=$V timeout 300 python scripts/prof_tc.py c4 2 > gpurun_out/${T}_c4_${V:-ch256}.log 2>&1
done
echo done
