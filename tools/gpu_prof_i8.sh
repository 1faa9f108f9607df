#!/bin/bash
# ncu --set full of the INT8 digit GEMMs (cuBLASLt) of the FP64 cross products.
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-tf32"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -k regex:"i256x256x32gemm_s8" -c 14 -o gpurun_out/prof_i8 $CMD > gpurun_out/ncu_i8.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_i8.log
