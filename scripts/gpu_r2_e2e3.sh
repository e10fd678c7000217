#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
rm -f gpurun_out/r2_e2e_sweep3.txt
for cfg in "GT_H2D=kernel PREFETCH_AT=build GT_H2D_CTAS=16" "GT_H2D=kernel PREFETCH_AT=build GT_H2D_CTAS=20" "GT_H2D=kernel PREFETCH_AT=start GT_H2D_CTAS=16" "GT_H2D=kernel PREFETCH_AT=start GT_H2D_CTAS=32" "GT_H2D=dma PREFETCH_AT=start" "GT_H2D=kernel PREFETCH_AT=build GT_H2D_CTAS=16"; do
  echo "== $cfg" >> gpurun_out/r2_e2e_sweep3.txt
  env $cfg timeout 300 python scripts/probe_e2e.py c4 2>&1 | tail -3 >> gpurun_out/r2_e2e_sweep3.txt
done
echo done
