# ncu --set full of the TC setup kernels (C2, step-only bench)
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-tsv --no-extras"
for k in cand_degree_kernel fill_rows_kernel place_tiles_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/full_tcs_$k $B > gpurun_out/ncu_tcs_$k.log 2>&1
  echo $k=$?
  ncu -i gpurun_out/full_tcs_$k.ncu-rep --page source --csv --print-source sass > gpurun_out/src_tcs_$k.csv 2>/dev/null
  ncu -i gpurun_out/full_tcs_$k.ncu-rep --page details > gpurun_out/det_tcs_$k.txt 2>/dev/null
done
