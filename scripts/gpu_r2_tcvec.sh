#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q tests/test_triangles_gpu.py -m gpu > gpurun_out/r2_tcvec_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2_tcvec_tests.log
rm -f gpurun_out/r2_tcvec.log
for v in 1 0; do
  echo "== GT_TC_VEC16=$v" >> gpurun_out/r2_tcvec.log
  GT_TC_VEC16=$v timeout 300 python scripts/prof_tc.py c4 2 2>&1 | grep -A3 "rep 1" >> gpurun_out/r2_tcvec.log
  GT_TC_VEC16=$v timeout 300 python scripts/prof_tc.py c2 3 2>&1 | grep -A2 "rep 2" >> gpurun_out/r2_tcvec.log
done
echo done
