#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q tests/test_build_gpu.py tests/test_bucket_build_gpu.py -m gpu > gpurun_out/r2_build_tests4.log 2>&1
echo "rc=$?" >> gpurun_out/r2_build_tests4.log
timeout 300 python scripts/prof_build.py c4 2 > gpurun_out/r2_prof_build_c4_v4.log 2>&1
timeout 300 python scripts/prof_build.py c2 3 > gpurun_out/r2_prof_build_c2_v4.log 2>&1
for v in default t4096 t1024 hot17 hot12; do
  if [ $v = default ]; then unset GT_LIB_VARIANT; else export GT_LIB_VARIANT=$v; fi
  echo "== $v" >> gpurun_out/r2_pr_sweep.log
  timeout 300 python scripts/prof_pagerank.py c4 2 2>&1 | grep -A3 "rep 1" >> gpurun_out/r2_pr_sweep.log
  timeout 300 python scripts/prof_pagerank.py c2 3 2>&1 | grep -A2 "rep 2" >> gpurun_out/r2_pr_sweep.log
done
unset GT_LIB_VARIANT
echo done
