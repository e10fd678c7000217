# usage: bash scripts/gpu_profile_set.sh <tag>  -- launch list + ncu --set full of the top kernels (C2 bench)
set -x
mkdir -p gpurun_out
TAG=${1:-cur}
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$B > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $B > gpurun_out/ncu_l_$TAG.log 2>&1
for k in tc_count_warp_kernel onesweep_kernel pr_spmv_kernel fill_rows_kernel place_rows_kernel cand_degree_kernel segment_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o gpurun_out/full_${TAG}_$k $B > gpurun_out/ncu_${TAG}_$k.log 2>&1
  echo $k=$?
done
