#!/bin/bash
# Per-sweep time vs the sweep grid (tiles per CTA, ENMF_SWEEP_TPC) at the column counts a rank
# sees when C5 is sharded over 8 / 4 GPUs (4096 / 8192), at C5 itself, and at the C1 / C2 shapes.
mkdir -p gpurun_out
for cfg in "128 4096" "128 8192" "128 32768" "40 400" "40 10304" "20 200"; do
  set -- $cfg
  for tpc in 16 4 2 1; do
    echo "r=$1 N=$2 tpc=$tpc $(SWEEP_R=$1 SWEEP_N=$2 ENMF_SWEEP_TPC=$tpc ENMF_SWEEP_FORCE=1 SWEEP_LONG=264 timeout 300 python tools/sweep_bench.py | tail -1)"
  done
done > gpurun_out/sweep_grid.txt 2>&1
