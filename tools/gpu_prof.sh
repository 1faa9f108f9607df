#!/bin/bash
# ncu captures of the dominant kernels (direct launches of e(0) and the profiled steps).
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:${SWEEP_RE:-sweep_dmma_p} -s 5 -c 1 -o gpurun_out/prof_sweep $CMD > gpurun_out/ncu_sweep.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_f64_dmma -s 1 -c 1 -o gpurun_out/prof_gemm1 $CMD > gpurun_out/ncu_gemm.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_gemm.log
