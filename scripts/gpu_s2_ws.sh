#!/bin/bash
# warp-specialised look-back sort kernel: parity (GT_SORT_PIPE=3) + C4 build timings
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
T=${1:-s2ws}
GT_SORT_PIPE=3 timeout 600 python -m pytest -x -q tests/test_build_gpu.py -m gpu > gpurun_out/${T}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
for V in "" ws3; do
  for P in 1 3; do
    GT_SORT_DEBUG=1 GT_LIB_VARIANT=$V GT_SORT_PIPE=$P timeout 300 python scripts/prof_build.py c4 2 > gpurun_out/${T}_${V:-base}_k$P.log 2>&1
  done
done
GT_SORT_DEBUG=1 GT_LIB_VARIANT=ws3lb2 GT_SORT_PIPE=1 timeout 300 python scripts/prof_build.py c4 2 > gpurun_out/${T}_ws3lb2_k1.log 2>&1
GT_SORT_PIPE=3 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^onesweep" -s 3 -c 1 -o gpurun_out/${T}_k3 python scripts/prof_build.py c4 1 > gpurun_out/${T}_ncu.log 2>&1
echo done
