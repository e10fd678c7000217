# Tuning sweep: radix-sort keys/thread ranked by __match_any_sync (GT_SORT_MATCH)
mkdir -p gpurun_out
for m in 0 6 8 11 16; do
  GT_SORT_MATCH=$m python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/bench_m$m.log 2>&1
  echo "m=$m $(python scripts/bench_summary.py gpurun_out/bench_m$m.log | grep -E 'out_sort|in_sort|tc.sort' | tr -s ' ' | tr '\n' ' ')"
done
