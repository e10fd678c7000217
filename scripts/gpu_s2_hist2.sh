#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
T=${1:-s2hist2}
timeout 900 python -m pytest -x -q tests/test_build_gpu.py tests/test_distributed_gpu.py tests/test_export_gpu.py tests/test_update_gpu.py tests/test_triangles_gpu.py::test_c2_c3_full_size_vs_oracles -m gpu > gpurun_out/${T}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
timeout 300 python scripts/prof_build.py c4 3 > gpurun_out/${T}_c4.log 2>&1
timeout 300 python scripts/prof_build.py c5 2 > gpurun_out/${T}_c5.log 2>&1
echo done
