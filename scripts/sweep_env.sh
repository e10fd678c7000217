# usage: bash scripts/sweep_env.sh <VAR> "v1 v2 ..." [bench args]  -- one bench per value of env VAR (no rebuild)
mkdir -p gpurun_out
N=$1; VALS=$2; shift 2
for V in $VALS; do
  env $N=$V timeout 900 python bench.py --no-e2e --no-cpu-baseline --no-tsv "$@" > gpurun_out/swe_${N}_$V.log 2>&1
  echo $N=$V rc=$?
  python scripts/bench_summary.py gpurun_out/swe_${N}_$V.log 2>/dev/null | head -12
done
