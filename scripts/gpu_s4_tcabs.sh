#!/bin/bash
# absolute-index, unchecked bitmap probes in the triangle count kernels: parity, then C4 / C2 timing
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
T=${1:-s4abs}
timeout 1200 python -m pytest -x -q tests/test_triangles_gpu.py tests/test_distributed_gpu.py tests/test_c_abi.py -m gpu > gpurun_out/${T}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
timeout 400 python scripts/prof_tc.py c4 2 > gpurun_out/${T}_c4.log 2>&1
timeout 400 python scripts/prof_tc.py c2 3 > gpurun_out/${T}_c2.log 2>&1
timeout 1500 python -m pytest -x -q tests/test_large_gpu.py tests/test_build_gpu.py -m gpu -k "triangle or c4 or c2_c3 or c3" > gpurun_out/${T}_pytest_large.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${T}_pytest_large.log
echo done
