# usage: bash scripts/sweep_const.sh <file> <NAME> "v1 v2 ..." [bench args]  -- rebuild per value of `constexpr int NAME`, one bench each
mkdir -p gpurun_out
F=$1; N=$2; VALS=$3; shift 3
cp $F /tmp/sweep_orig
for V in $VALS; do
  sed -e "s/^constexpr int $N = [0-9]*;/constexpr int $N = $V;/" /tmp/sweep_orig > $F
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_${N}_$V.log 2>&1 || { echo build $V failed; continue; }
  python bench.py --no-e2e --no-cpu-baseline --no-tsv "$@" > gpurun_out/sw_${N}_$V.log 2>&1
  echo $N=$V rc=$?
done
cp /tmp/sweep_orig $F
