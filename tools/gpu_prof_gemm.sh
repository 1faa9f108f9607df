#!/bin/bash
# ncu --set full of the first few FP64 DMMA GEMM launches of a short bench (the large
# W_yᵀX / X·Tᵀ products are among them; pick by grid size when reading).
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:gemm_f64_dmma_s -c ${COUNT:-4} -o gpurun_out/prof_gemm_s $CMD > gpurun_out/ncu_gemm.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_gemm.log
