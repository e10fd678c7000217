#!/bin/bash
# PageRank: push within L2-sized destination bins vs the pull SpMV
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
T=${1:-s2push}
GT_PR_PUSH=1 timeout 900 python -m pytest -x -q tests/test_pagerank_gpu.py -m gpu -k "not determinism" > gpurun_out/${T}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
for C in c4 c5 c2; do
  for P in 0 1; do
    GT_PR_PUSH=$P timeout 400 python scripts/prof_pagerank.py $C 2 > gpurun_out/${T}_${C}_p$P.log 2>&1
  done
done
echo done
