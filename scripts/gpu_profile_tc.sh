# usage: bash scripts/gpu_profile_tc.sh <tag>  -- ncu --set full of the TC kernels (one launch per step: skip the warm-up launch)
mkdir -p gpurun_out
TAG=${1:-cur}
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-tsv"
for k in tc_count_warp_kernel fill_rows_kernel place_rows_kernel cand_degree_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/full_${TAG}_$k $B > gpurun_out/ncu_${TAG}_$k.log 2>&1
  echo $k=$?
done
