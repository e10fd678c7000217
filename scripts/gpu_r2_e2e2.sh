#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
rm -f gpurun_out/r2_e2e_sweep2.txt
for c in 4 6 8 12 24; do
  echo "== kernel build CTAS=$c" >> gpurun_out/r2_e2e_sweep2.txt
  GT_H2D=kernel PREFETCH_AT=build GT_H2D_CTAS=$c timeout 300 python scripts/probe_e2e.py c4 2>&1 | tail -2 >> gpurun_out/r2_e2e_sweep2.txt
done
echo done
