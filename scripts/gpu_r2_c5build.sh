#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
GT_BK_STATS=1 timeout 400 python scripts/prof_build.py c5 2 > gpurun_out/r2_prof_build_c5_bucket.log 2>&1
GT_BUILD=sort timeout 400 python scripts/prof_build.py c5 2 > gpurun_out/r2_prof_build_c5_sort.log 2>&1
GT_BUILD=sort timeout 400 python scripts/prof_build.py c4 2 > gpurun_out/r2_prof_build_c4_sort.log 2>&1
echo done
