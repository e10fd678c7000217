#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
T=${1:-s2pipe3}
timeout 600 python -m pytest -x -q tests/test_build_gpu.py -m gpu > gpurun_out/${T}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
GT_SORT_PIPE=1 timeout 300 python scripts/prof_build.py c4 2 > gpurun_out/${T}_build_c4_pipe1.log 2>&1
GT_SORT_PIPE=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^onesweep_pipe" -s 3 -c 1 -o gpurun_out/${T}_pipe python scripts/prof_build.py c4 1 > gpurun_out/${T}_ncu.log 2>&1
echo done
