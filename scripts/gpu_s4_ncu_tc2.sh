#!/bin/bash
# full ncu captures (with source) of the CTA count kernel and the orientation kernels at C4
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
T=${1:-s4tc2}
for K in tc_count_cta_kernel place_tiles_kernel fill_rows_kernel cand_degree_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 \
    -o gpurun_out/${T}_$K python scripts/prof_tc.py c4 2 > gpurun_out/${T}_ncu_$K.log 2>&1
done
echo done
