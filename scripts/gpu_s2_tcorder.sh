#!/bin/bash
# bitmap triangle tasks in u order vs v order: parity + C4/C2 timings
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
T=${1:-s2tco}
timeout 900 python -m pytest -x -q tests/test_triangles_gpu.py -m gpu > gpurun_out/${T}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
for O in 0 1; do
  GT_TC_ORDER=$O timeout 300 python scripts/prof_tc.py c4 2 > gpurun_out/${T}_c4_o$O.log 2>&1
  GT_TC_ORDER=$O timeout 300 python scripts/prof_tc.py c2 3 > gpurun_out/${T}_c2_o$O.log 2>&1
done
echo done
