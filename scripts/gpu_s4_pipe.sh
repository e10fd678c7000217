#!/bin/bash
# Pipelined PageRank pull (GT_PR_PIPE=1): parity tests, C4 / C2 timing A/B, ncu counters.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
T=${1:-s4pipe}
GT_PR_PIPE=1 timeout 900 python -m pytest -x -q tests/test_pagerank_gpu.py -m gpu > gpurun_out/${T}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
for P in 0 1; do
  GT_PR_DEBUG=1 GT_PR_PIPE=$P timeout 400 python scripts/prof_pagerank.py c4 2 > gpurun_out/${T}_c4_p$P.log 2>&1
  GT_PR_PIPE=$P timeout 400 python scripts/prof_pagerank.py c2 3 > gpurun_out/${T}_c2_p$P.log 2>&1
done
GT_PR_PIPE=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:pr_spmv_pipe -s 22 -c 1 \
  -o gpurun_out/${T}_pr_pipe python scripts/prof_pagerank.py c4 2 > gpurun_out/${T}_ncu.log 2>&1
echo done
