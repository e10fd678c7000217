#!/bin/bash
# triangle count walk constants (build knobs) at C4 and C2
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
T=${1:-s4var}
for V in base cc8k cc32k c128 c512; do
  if [ "$V" = base ]; then unset GT_LIB_VARIANT; else export GT_LIB_VARIANT=$V; fi
  timeout 400 python scripts/prof_tc.py c4 2 2>&1 | grep -E "^rep 1|tc.count" | tail -3 > gpurun_out/${T}_c4_$V.log
  timeout 400 python scripts/prof_tc.py c2 3 2>&1 | grep -E "^rep 2|tc.count" | tail -2 > gpurun_out/${T}_c2_$V.log
done
echo done
