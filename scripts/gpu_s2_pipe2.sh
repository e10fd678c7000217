#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
T=${1:-s2pipe2}
GT_SORT_DEBUG=1 GT_SORT_PIPE=1 timeout 300 python scripts/prof_build.py c4 2 > gpurun_out/${T}_build_c4_pipe1.log 2>&1
for K in onesweep_kernel onesweep_pipe_kernel; do
  P=1; [ $K = onesweep_kernel ] && P=0
  GT_SORT_PIPE=$P timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^$K" -s 3 -c 1 -o gpurun_out/${T}_$K python scripts/prof_build.py c4 1 > gpurun_out/${T}_ncu_$K.log 2>&1
done
echo done
