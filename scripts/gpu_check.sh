# usage: bash scripts/gpu_check.sh [pytest -k expr]  -- tests + smoke + bench on one B200
set -x
mkdir -p gpurun_out
K=${1:-}
if [ -n "$K" ]; then timeout 900 python -m pytest tests -x -q -m gpu -k "$K" > gpurun_out/pytest_gpu.log 2>&1; else timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; fi
echo pytest=$?
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
tail -2 gpurun_out/smoke.log
timeout 600 python bench.py ${BENCH_ARGS:---steps 3 --warmup 3} > gpurun_out/bench.log 2>&1; echo bench=$?
tail -c 3000 gpurun_out/bench.log
