#!/bin/bash
# Session 4: L2 prefetch of the tile one residency wave ahead (sort passes,
# PageRank index stream) A/B at C4, then one full ncu capture of pr_spmv.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
T=${1:-s4pf}
timeout 600 python -m pytest -x -q tests/test_build_gpu.py tests/test_pagerank_gpu.py -m gpu > gpurun_out/${T}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
for P in 0 296 592 1184 2368; do
  GT_SORT_PF=$P timeout 400 python scripts/prof_build.py c4 3 2>&1 | grep -E "rep 2|out_sort|in_sort" | tail -3 > gpurun_out/${T}_sort_pf$P.log
done
for P in 0 444 888 1776 3552; do
  GT_PR_PF=$P timeout 400 python scripts/prof_pagerank.py c4 2 2>&1 | grep -E "rep 1|pr.spmv" | tail -2 > gpurun_out/${T}_pr_pf$P.log
done
timeout 900 ncu --set full --clock-control none --import-source on -k pr_spmv_kernel -s 22 -c 1 \
  -o gpurun_out/${T}_pr_spmv python scripts/prof_pagerank.py c4 2 > gpurun_out/${T}_ncu_pr.log 2>&1
echo done
