#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
T=${1:-s2dist}
timeout 900 python -m pytest -x -q tests/test_distributed_gpu.py tests/test_triangles_gpu.py tests/test_native_abi.py tests/test_c_abi.py -m gpu > gpurun_out/${T}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
timeout 600 python bench.py --config c2 --no-extras --sharded --steps 3 --warmup 3 > gpurun_out/${T}_bench_c2_sharded.json 2> gpurun_out/${T}_bench_c2_sharded.err
echo done
