#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
T=${1:-r2f}
timeout 900 python bench.py > gpurun_out/${T}_bench_c4.json 2> gpurun_out/${T}_bench_c4.err
timeout 600 python bench.py --config c2 > gpurun_out/${T}_bench_c2.json 2> gpurun_out/${T}_bench_c2.err
timeout 900 python bench.py --config c5 --no-extras > gpurun_out/${T}_bench_c5.json 2> gpurun_out/${T}_bench_c5.err
timeout 900 python bench.py --impl reference > gpurun_out/${T}_bench_ref_c4.json 2> gpurun_out/${T}_bench_ref_c4.err
echo done
