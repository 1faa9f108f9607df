#!/bin/bash
# Sweep-kernel timing (tools/sweep_bench.py) for a few variants + the ws per-warp cycle profiles.
mkdir -p gpurun_out
for v in ${VARIANTS:-ws t14u2}; do
  ENMF_HALS_KERNEL=$v timeout 120 python tools/sweep_bench.py >> gpurun_out/sweep_bench.log 2>&1
done
for v in ${PROFS:-wsprof wsprof1 wsprof2}; do
  echo "== $v" >> gpurun_out/sweep_bench.log
  ENMF_HALS_KERNEL=$v ENMF_SWEEP_PROF=1 timeout 120 python tools/sweep_bench.py 2>&1 | tail -3 >> gpurun_out/sweep_bench.log
done
echo done >> gpurun_out/sweep_bench.log
