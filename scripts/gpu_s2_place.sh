#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
T=${1:-s2pl}
timeout 900 python -m pytest -x -q tests/test_triangles_gpu.py -m gpu > gpurun_out/${T}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
for V in "" pdirect; do
  GT_LIB_VARIANT=$V timeout 300 python scripts/prof_tc.py c4 2 > gpurun_out/${T}_c4_${V:-agg}.log 2>&1
done
echo done
