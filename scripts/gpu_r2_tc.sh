#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
GT_TC_STATS=1 timeout 300 python scripts/prof_tc.py c4 2 > gpurun_out/r2_prof_tc_c4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_count -s 2 -c 2 -o gpurun_out/r2_tc_c4 python scripts/prof_tc.py c4 2 > gpurun_out/r2_ncu_tc.log 2>&1
echo done
