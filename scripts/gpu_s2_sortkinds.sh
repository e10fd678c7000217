#!/bin/bash
# parity of the default sort kernel + C4 build timings for every GT_SORT_PIPE kind
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
T=${1:-s2kinds}
timeout 600 python -m pytest -x -q tests/test_build_gpu.py -m gpu > gpurun_out/${T}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
for P in 0 1 2; do
  GT_SORT_DEBUG=1 GT_SORT_PIPE=$P timeout 300 python scripts/prof_build.py c4 2 > gpurun_out/${T}_build_c4_k$P.log 2>&1
done
if [ -n "$NCU_KIND" ]; then
GT_SORT_PIPE=$NCU_KIND timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^onesweep" -s 3 -c 1 -o gpurun_out/${T}_k$NCU_KIND python scripts/prof_build.py c4 1 > gpurun_out/${T}_ncu.log 2>&1
fi
echo done
