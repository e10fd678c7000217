#!/bin/bash
# shared-memory-ranked sort kernel: 256- vs 512-thread CTAs, look-back window 2 vs 4
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
T=${1:-s2nt}
GT_SORT_KERNEL=2 timeout 600 python -m pytest -x -q tests/test_build_gpu.py -m gpu > gpurun_out/${T}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
for V in "" slb4; do
  for P in 1 2; do
    GT_SORT_DEBUG=1 GT_LIB_VARIANT=$V GT_SORT_KERNEL=$P timeout 300 python scripts/prof_build.py c4 2 > gpurun_out/${T}_${V:-base}_k$P.log 2>&1
  done
done
echo done
