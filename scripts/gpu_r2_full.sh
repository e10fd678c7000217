#!/bin/bash
# full GPU suite + default bench (the driver's round-end commands) + reference arm
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
T=${1:-r2}
timeout 1800 python -m pytest tests -x -q -m gpu --durations=15 > gpurun_out/${T}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/${T}_smoke.log
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
echo "bench rc=$?" >> gpurun_out/${T}_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/${T}_bench_ref.json 2> gpurun_out/${T}_bench_ref.err
echo "ref rc=$?" >> gpurun_out/${T}_bench_ref.err
echo done
