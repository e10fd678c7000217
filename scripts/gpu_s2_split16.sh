#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
T=${1:-s2sp}
timeout 1200 python -m pytest -x -q tests/test_triangles_gpu.py tests/test_distributed_gpu.py tests/test_large_gpu.py::test_c4_triangle_slice_vs_oracle -m gpu > gpurun_out/${T}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
timeout 300 python scripts/prof_tc.py c4 2 > gpurun_out/${T}_c4.log 2>&1
timeout 300 python scripts/prof_tc.py c2 3 > gpurun_out/${T}_c2.log 2>&1
echo done
