#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1500 python -m pytest -x -q tests/test_reference_suite_gpu.py tests/test_large_gpu.py -m gpu > gpurun_out/r2_subset2.log 2>&1
echo "rc=$?" >> gpurun_out/r2_subset2.log
cp gpurun_out/reference_suite_on_dropin.log gpurun_out/r2_reference_suite.log 2>/dev/null
echo done
