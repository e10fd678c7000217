#!/bin/bash
# A/B of the pipelined (bulk-copy, persistent) onesweep pass vs the
# one-tile-per-CTA pass: parity tests with the new default, then C4/C5 build timings.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
T=${1:-s2pipe}
timeout 900 python -m pytest -x -q tests/test_build_gpu.py tests/test_update_gpu.py tests/test_triangles_gpu.py::test_c2_c3_full_size_vs_oracles -m gpu > gpurun_out/${T}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
for P in 0 1; do
  GT_SORT_PIPE=$P timeout 300 python scripts/prof_build.py c4 3 > gpurun_out/${T}_build_c4_pipe$P.log 2>&1
done
GT_SORT_PIPE=1 timeout 300 python scripts/prof_build.py c5 2 > gpurun_out/${T}_build_c5_pipe1.log 2>&1
echo done
