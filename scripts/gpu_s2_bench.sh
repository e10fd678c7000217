#!/bin/bash
# default bench (the driver's command) + C2 line
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
T=${1:-s2b}
timeout 900 python bench.py > gpurun_out/${T}_bench_c4.json 2> gpurun_out/${T}_bench_c4.err
echo "bench rc=$?" >> gpurun_out/${T}_bench_c4.err
timeout 600 python bench.py --config c2 --no-extras > gpurun_out/${T}_bench_c2.json 2> gpurun_out/${T}_bench_c2.err
echo done
