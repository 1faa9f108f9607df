#!/bin/bash
# ncu --set full capture of one HALS sweep launch (SWEEP_RE selects the kernel).
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${SWEEP_RE:-sweep_ws} -s 20 -c 1 -o gpurun_out/prof_sweep $CMD > gpurun_out/ncu_sweep.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_sweep.log
