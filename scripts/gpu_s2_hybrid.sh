#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
T=${1:-s2hy}
timeout 900 python -m pytest -x -q tests/test_pagerank_gpu.py -m gpu > gpurun_out/${T}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
for P in 0 2; do
  GT_PR_PUSH=$P timeout 400 python scripts/prof_pagerank.py c4 2 > gpurun_out/${T}_c4_p$P.log 2>&1
done
timeout 400 python scripts/prof_pagerank.py c4 2 > gpurun_out/${T}_c4_auto.log 2>&1
echo done
