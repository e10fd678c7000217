# ncu --set full of the dominant kernels at C4 (one launch each, step-only bench)
mkdir -p gpurun_out
B="python bench.py --config c4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-tsv --no-extras"
for k in pr_spmv_kernel onesweep_kernel tc_count_warp_kernel; do
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o gpurun_out/full_c4_$k $B > gpurun_out/ncu_c4_$k.log 2>&1
  echo $k=$?
done
