#!/bin/bash
# in-sort histograms folded from the out-sort's: parity + C4/C2 build timings
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
T=${1:-s2hist}
timeout 900 python -m pytest -x -q tests/test_build_gpu.py tests/test_distributed_gpu.py tests/test_export_gpu.py tests/test_triangles_gpu.py::test_c2_c3_full_size_vs_oracles -m gpu > gpurun_out/${T}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
for V in "" lbsync; do
  GT_LIB_VARIANT=$V timeout 300 python scripts/prof_build.py c4 3 > gpurun_out/${T}_${V:-base}_c4.log 2>&1
done
timeout 300 python scripts/prof_build.py c2 3 > gpurun_out/${T}_base_c2.log 2>&1
echo done
