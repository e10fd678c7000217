# usage: bash scripts/gpu_profile_v4b.sh -- step-only launch lists (C2, C4) + ncu --set full of the TC kernels
set -x
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-tsv --no-extras"
$B > gpurun_out/plain_v4b.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v4_c2.csv $B > gpurun_out/ncu_l_v4b.log 2>&1; echo launches_c2=$?
B4="python bench.py --config c4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-tsv --no-extras"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v4_c4.csv $B4 > gpurun_out/ncu_l_v4c4.log 2>&1; echo launches_c4=$?
for k in tc_count_warp_kernel place_tiles_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/full_v4_$k $B > gpurun_out/ncu_v4_$k.log 2>&1
  echo $k=$?
done
