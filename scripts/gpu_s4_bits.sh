#!/bin/bash
# 9-bit radix digits for the two big sorts of the build (GT_SORT_BITS=9 vs 8): parity, then C4 / C2 / C5 timing.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
T=${1:-s4bits}
GT_SORT_BITS=9 timeout 1200 python -m pytest -x -q tests/test_build_gpu.py tests/test_bucket_build_gpu.py tests/test_c_abi.py tests/test_distributed_gpu.py tests/test_update_gpu.py -m gpu > gpurun_out/${T}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
for B in 8 9; do
  GT_SORT_DEBUG=1 GT_SORT_BITS=$B timeout 400 python scripts/prof_build.py c4 3 > gpurun_out/${T}_c4_b$B.log 2>&1
  GT_SORT_BITS=$B timeout 400 python scripts/prof_build.py c2 3 > gpurun_out/${T}_c2_b$B.log 2>&1
  GT_SORT_BITS=$B timeout 400 python scripts/prof_build.py c5 3 > gpurun_out/${T}_c5_b$B.log 2>&1
done
GT_SORT_BITS=9 timeout 1500 python -m pytest -x -q tests/test_large_gpu.py -m gpu > gpurun_out/${T}_pytest_large.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${T}_pytest_large.log
echo done
