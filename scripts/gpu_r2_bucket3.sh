#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_bucket_build_gpu.py -x -q > gpurun_out/r2_bk_tests3.log 2>&1
echo "bucket tests rc=$?" >> gpurun_out/r2_bk_tests3.log
GT_BK_STATS=1 timeout 300 python scripts/prof_build.py c4 3 > gpurun_out/r2_prof_build_c4_v3.log 2>&1
GT_BK_STATS=1 timeout 300 python scripts/prof_build.py c2 3 > gpurun_out/r2_prof_build_c2_v3.log 2>&1
timeout 900 python -m pytest tests/test_build_gpu.py -x -q > gpurun_out/r2_build_tests3.log 2>&1
echo "build tests rc=$?" >> gpurun_out/r2_build_tests3.log
echo done
