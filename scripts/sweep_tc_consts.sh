# usage: bash scripts/sweep_tc_consts.sh "LONG:WIN:UNROLL ..."  -- rebuild per combination, one C2 bench each
mkdir -p gpurun_out
F=paper_1503_07881_b200/csrc/triangles.cu
cp $F /tmp/tri_orig.cu
for C in $1; do
  IFS=: read L W U <<< "$C"
  sed -e "s/^constexpr int TC_LONG = [0-9]*;/constexpr int TC_LONG = $L;/" \
      -e "s/^constexpr int TC_WIN = [0-9]*;/constexpr int TC_WIN = $W;/" \
      -e "s/^constexpr int TC_UNROLL = [0-9]*;/constexpr int TC_UNROLL = $U;/" /tmp/tri_orig.cu > $F
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$C.log 2>&1 || { echo build $C failed; continue; }
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-tsv > gpurun_out/tcc_$C.log 2>&1
  echo C=$C rc=$?
done
cp /tmp/tri_orig.cu $F
