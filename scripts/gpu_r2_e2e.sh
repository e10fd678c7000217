#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
rm -f gpurun_out/r2_e2e_sweep.txt
for cfg in "GT_H2D=dma PREFETCH_AT=build" "GT_H2D=dma PREFETCH_AT=tc" "GT_H2D=kernel PREFETCH_AT=tc GT_H2D_CTAS=32" "GT_H2D=kernel PREFETCH_AT=tc GT_H2D_CTAS=16" "GT_H2D=kernel PREFETCH_AT=tc GT_H2D_CTAS=64" "GT_H2D=kernel PREFETCH_AT=build GT_H2D_CTAS=16"; do
  echo "== $cfg" >> gpurun_out/r2_e2e_sweep.txt
  env $cfg timeout 300 python scripts/probe_e2e.py c4 2>&1 | tail -2 >> gpurun_out/r2_e2e_sweep.txt
done
echo done
