set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python bench.py --steps 3 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench=$?
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$B > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu1.log 2>&1; echo ncu1=$?
for k in tc_count_kernel onesweep_kernel pr_spmv_kernel segment_kernel; do
ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o gpurun_out/prof_$k $B > gpurun_out/ncu_$k.log 2>&1; echo $k=$?
done
