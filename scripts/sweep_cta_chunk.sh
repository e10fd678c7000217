# usage: bash scripts/sweep_cta_chunk.sh "1024 4096"  -- rebuild per TC_CHUNK_CTA, one C4 bench each
mkdir -p gpurun_out
F=paper_1503_07881_b200/csrc/triangles.cu
cp $F /tmp/tri_orig.cu
for C in $1; do
  sed -e "s/^constexpr int TC_CHUNK_CTA = [0-9]*;/constexpr int TC_CHUNK_CTA = $C;/" /tmp/tri_orig.cu > $F
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_cc$C.log 2>&1 || { echo build $C failed; continue; }
  python bench.py --config c4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-tsv > gpurun_out/cc_$C.log 2>&1
  echo C=$C rc=$?
done
cp /tmp/tri_orig.cu $F
