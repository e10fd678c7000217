#!/bin/bash
# Session-4 PageRank probes at C4: evict_last head size sweep, policy off, and
# per-launch ncu counters (the last iteration writes scores sequentially, the
# others scatter contrib_next: their difference prices the scatter).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
T=${1:-s4pr}
GT_PR_DEBUG=1 timeout 400 python scripts/prof_pagerank.py c4 2 > gpurun_out/${T}_default.log 2>&1
for H in 8 16 32 48 64 96; do
  GT_PR_HOT_MB=$H timeout 400 python scripts/prof_pagerank.py c4 2 2>&1 | grep -E "rep 1|pr.spmv" > gpurun_out/${T}_hot$H.log
done
GT_PR_L2=none timeout 400 python scripts/prof_pagerank.py c4 2 2>&1 | grep -E "rep 1|pr.spmv" > gpurun_out/${T}_l2none.log
timeout 900 ncu --cache-control none --clock-control none \
  --metrics gpu__time_duration.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  -k pr_spmv_kernel -c 20 --csv --log-file gpurun_out/${T}_ncu_launches.csv \
  python scripts/prof_pagerank.py c4 1 > gpurun_out/${T}_ncu.log 2>&1
echo done
