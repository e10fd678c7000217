#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
T=${1:-s2push2}
timeout 1500 python -m pytest -x -q tests/test_pagerank_gpu.py tests/test_large_gpu.py -m gpu > gpurun_out/${T}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
for C in c5 c4; do
  timeout 400 python scripts/prof_pagerank.py $C 2 > gpurun_out/${T}_${C}_auto.log 2>&1
done
echo done
