#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q tests/test_triangles_gpu.py -m gpu > gpurun_out/r2_tc_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2_tc_tests.log
rm -f gpurun_out/r2_tc_sweep.log
for v in default bm6 bm4c4k bm6c1k; do
  if [ $v = default ]; then unset GT_LIB_VARIANT; else export GT_LIB_VARIANT=$v; fi
  echo "== $v" >> gpurun_out/r2_tc_sweep.log
  timeout 300 python scripts/prof_tc.py c4 2 2>&1 | grep -A4 "rep 1" >> gpurun_out/r2_tc_sweep.log
  timeout 300 python scripts/prof_tc.py c2 3 2>&1 | grep -A3 "rep 2" >> gpurun_out/r2_tc_sweep.log
done
echo done
