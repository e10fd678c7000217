#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_bucket_build_gpu.py -x -q > gpurun_out/r2_bk_tests2.log 2>&1
echo "bucket tests rc=$?" >> gpurun_out/r2_bk_tests2.log
GT_BK_STATS=1 timeout 300 python scripts/prof_build.py c4 3 > gpurun_out/r2_prof_build_c4.log 2>&1
GT_BK_STATS=1 timeout 300 python scripts/prof_build.py c2 3 > gpurun_out/r2_prof_build_c2.log 2>&1
timeout 300 python scripts/prof_build.py c4 2 > gpurun_out/r2_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bk_leaf_kernel -s 2 -c 2 -o gpurun_out/r2_leaf_c4 python scripts/prof_build.py c4 2 > gpurun_out/r2_ncu_leaf.log 2>&1
echo done
