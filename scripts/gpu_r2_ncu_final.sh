#!/bin/bash
# round-2 evidence at C4: bench launch list, per-kernel DRAM bytes of the
# build and of PageRank, one full capture of the dominant HBM kernel
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --no-extras --no-e2e --no-cpu-baseline"
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
$B > gpurun_out/r2n_bench_plain.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2n_launches_c4.csv $B > gpurun_out/r2n_ncu_launch.log 2>&1
python scripts/prof_build.py c4 1 > gpurun_out/r2n_build_plain.log 2>&1 && \
timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r2n_build_dram_c4.csv python scripts/prof_build.py c4 1 > gpurun_out/r2n_ncu_build.log 2>&1
python scripts/prof_pagerank.py c4 1 > gpurun_out/r2n_pr_plain.log 2>&1 && \
timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r2n_pr_dram_c4.csv python scripts/prof_pagerank.py c4 1 > gpurun_out/r2n_ncu_pr.log 2>&1
python scripts/prof_pagerank.py c4 1 > gpurun_out/r2n_pr_plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pr_spmv_kernel -s 5 -c 1 -o gpurun_out/r2n_full_c4_pr_spmv python scripts/prof_pagerank.py c4 1 > gpurun_out/r2n_ncu_full_pr.log 2>&1
echo done
