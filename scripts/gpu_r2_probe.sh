#!/bin/bash
# round-2 probe: host facts, design microbenchmarks, current C4 bench
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
{ nproc; free -g; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv; } > gpurun_out/r2_host.txt 2>&1
timeout 300 ./scripts/ubench/ubench_r2 part > gpurun_out/r2_ubench_part.txt 2>&1
timeout 300 ./scripts/ubench/ubench_r2 gather notma > gpurun_out/r2_ubench_gather.txt 2>&1
timeout 120 ./scripts/ubench/ubench_r2 gather > gpurun_out/r2_ubench_gather_tma.txt 2>&1
timeout 900 python bench.py --config c4 --steps 3 --warmup 2 --no-extras --no-cpu-baseline > gpurun_out/r2_bench_c4_v0.json 2> gpurun_out/r2_bench_c4_v0.err
echo done
