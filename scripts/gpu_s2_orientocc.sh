#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
T=${1:-s2oo}
for V in "" pl6 pl7 fi4 fi5; do
  GT_LIB_VARIANT=$V timeout 300 python scripts/prof_tc.py c4 2 > gpurun_out/${T}_c4_${V:-base}.log 2>&1
done
echo done
