# usage: bash scripts/gpu_profile_v4.sh  -- round-1 v4 evidence: C2 bench (full contract line), C4 bench,
# C2 launch list, ncu --set full of the top kernels
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r1_v4_bench_c2.log 2>&1; echo bench_c2=$?
timeout 900 python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline --no-tsv > gpurun_out/r1_v4_bench_c4.log 2>&1; echo bench_c4=$?
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-tsv"
$B > gpurun_out/plain_v4.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v4.csv $B > gpurun_out/ncu_l_v4.log 2>&1; echo launches=$?
for k in tc_count_warp_kernel onesweep_kernel pr_spmv_kernel place_tiles_kernel segment_kernel pack_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o gpurun_out/full_v4_$k $B > gpurun_out/ncu_v4_$k.log 2>&1
  echo $k=$?
done
