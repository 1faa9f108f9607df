#!/bin/bash
# Per-sweep time of the persistent HALS sweep at C5 with parts of the work switched off
# (wspprof1: no row pass, wspprof2: no DMMA products, wspprof3: neither) — timing only;
# ENMF_SWEEP_FORCE runs every sweep regardless of the stall rule.
mkdir -p gpurun_out
for v in ${VARIANTS:-wsp wspprof wspprof1 wspprof2 wspprof3}; do
  ENMF_SWEEP_FORCE=1 ENMF_SWEEP_PROF=1 SWEEP_LONG=264 ENMF_HALS_KERNEL=$v timeout 300 python tools/sweep_bench.py
done > gpurun_out/sweep_breakdown.txt 2>&1
