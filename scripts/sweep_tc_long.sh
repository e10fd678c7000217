# usage: bash scripts/sweep_tc_long.sh "16 48 128"  -- rebuild with each TC_LONG, one C2 bench each
mkdir -p gpurun_out
F=paper_1503_07881_b200/csrc/triangles.cu
cp $F /tmp/tri_orig.cu
for L in $1; do
  sed "s/^constexpr int TC_LONG = [0-9]*;/constexpr int TC_LONG = $L;/" /tmp/tri_orig.cu > $F
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$L.log 2>&1 || { echo build $L failed; continue; }
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-tsv > gpurun_out/long_$L.log 2>&1
  echo L=$L rc=$?
done
cp /tmp/tri_orig.cu $F
