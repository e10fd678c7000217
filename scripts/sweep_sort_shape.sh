# usage: bash scripts/sweep_sort_shape.sh "kpt:minblocks ..." [bench args] -- onesweep tile shape sweep (rebuild per point)
mkdir -p gpurun_out
PTS=$1; shift
H=paper_1503_07881_b200/csrc/radix_sort.cuh; C=paper_1503_07881_b200/csrc/radix_sort.cu
cp $H /tmp/sw_h; cp $C /tmp/sw_c
for P in $PTS; do
  K=${P%%:*}; M=${P##*:}
  sed -e "s/^constexpr int RS_KPT = [0-9]*;/constexpr int RS_KPT = $K;/" /tmp/sw_h > $H
  sed -e "s/^constexpr int RS_MIN_BLOCKS = [0-9]*;/constexpr int RS_MIN_BLOCKS = $M;/" /tmp/sw_c > $C
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_shape_$K_$M.log 2>&1 || { echo build $P failed; continue; }
  python bench.py --no-e2e --no-cpu-baseline --no-tsv "$@" > gpurun_out/sw_shape_${K}_$M.log 2>&1
  echo "shape $P rc=$?"
  python scripts/bench_summary.py gpurun_out/sw_shape_${K}_$M.log | grep -E "out_sort|in_sort"
done
cp /tmp/sw_h $H; cp /tmp/sw_c $C
