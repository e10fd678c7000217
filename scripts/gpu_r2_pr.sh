#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_pagerank_gpu.py -x -q > gpurun_out/r2_pr_tests.log 2>&1
echo "pr tests rc=$?" >> gpurun_out/r2_pr_tests.log
timeout 300 python scripts/prof_pagerank.py c4 2 > gpurun_out/r2_prof_pr_c4.log 2>&1
GT_PR_BLOCK=0 timeout 300 python scripts/prof_pagerank.py c4 2 > gpurun_out/r2_prof_pr_c4_single.log 2>&1
timeout 400 python scripts/prof_pagerank.py c5 2 > gpurun_out/r2_prof_pr_c5.log 2>&1
timeout 900 python -m pytest tests/test_large_gpu.py -x -q -k pagerank > gpurun_out/r2_pr_large.log 2>&1
echo "large rc=$?" >> gpurun_out/r2_pr_large.log
echo done
