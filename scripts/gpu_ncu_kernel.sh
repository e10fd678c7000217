# usage: bash scripts/gpu_ncu_kernel.sh <kernel-regex> [skip] [tag]  -- one ncu --set full capture of a bench kernel
set -x
mkdir -p gpurun_out
K=$1; S=${2:-0}; TAG=${3:-$1}
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$B > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 -o gpurun_out/prof_$TAG $B > gpurun_out/ncu_$TAG.log 2>&1
echo ncu=$?
tail -3 gpurun_out/ncu_$TAG.log
