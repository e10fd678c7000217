#!/bin/bash
# merge_runs parity + timing on one B200
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_distributed_gpu.py -x -q 2>&1 | tail -15 | tee gpurun_out/merge_tests.log
timeout 300 python scripts/prof_merge.py 2>&1 | tail -10 | tee gpurun_out/merge_prof.log
timeout 900 python bench.py > gpurun_out/bench_c4_after_prefetch.json 2> gpurun_out/bench_c4_after_prefetch.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench_c4_after_prefetch.json
