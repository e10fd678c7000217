#!/bin/bash
# round 2: bucket-build parity + first timing
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_bucket_build_gpu.py -x -q > gpurun_out/r2_bk_tests.log 2>&1
echo "bucket tests rc=$?" >> gpurun_out/r2_bk_tests.log
timeout 900 python -m pytest tests/test_build_gpu.py -x -q > gpurun_out/r2_build_tests.log 2>&1
echo "build tests rc=$?" >> gpurun_out/r2_build_tests.log
timeout 600 python bench.py --config c4 --steps 3 --warmup 2 --no-extras --no-cpu-baseline --no-e2e > gpurun_out/r2_bench_c4_v1.json 2> gpurun_out/r2_bench_c4_v1.err
echo done
