#!/bin/bash
# L2 hit counters of pr_spmv at C4 for several evict_last head sizes.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
T=${1:-s4hot}
for H in 8 16 32 48 79; do
  GT_PR_HOT_MB=$H timeout 600 ncu --cache-control none --clock-control none \
    --metrics gpu__time_duration.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_requests_srcunit_ltcfabric.sum,dram__bytes_read.sum \
    -k regex:pr_spmv_kernel -s 5 -c 2 --csv --log-file gpurun_out/${T}_h$H.csv \
    python scripts/prof_pagerank.py c4 1 > gpurun_out/${T}_h$H.log 2>&1
done
GT_PR_L2=none timeout 600 ncu --cache-control none --clock-control none \
    --metrics gpu__time_duration.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_requests_srcunit_ltcfabric.sum,dram__bytes_read.sum \
    -k regex:pr_spmv_kernel -s 5 -c 2 --csv --log-file gpurun_out/${T}_none.csv \
    python scripts/prof_pagerank.py c4 1 > gpurun_out/${T}_none.log 2>&1
echo done
for S in 10 12 13; do
  GT_PR_DEBUG=1 GT_PR_SHOT=$S GT_PR_PF=0 timeout 400 python scripts/prof_pagerank.py c4 2 2>&1 | grep -E "CTAs|rep 1|pr.spmv" | tail -3 > gpurun_out/${T}_shot$S.log
done
GT_PR_SHOT=12 timeout 600 python -m pytest -x -q tests/test_pagerank_gpu.py -m gpu > gpurun_out/${T}_pytest_shot.log 2>&1
echo done2
