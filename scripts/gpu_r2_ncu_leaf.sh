#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 300 python scripts/prof_build.py c4 2 > gpurun_out/r2_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bk_leaf_kernel -s 2 -c 2 -o gpurun_out/r2_leaf_c4_v5 python scripts/prof_build.py c4 2 > gpurun_out/r2_ncu_leaf5.log 2>&1
echo done
