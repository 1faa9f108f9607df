#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_f64_dmma -s 1 -c 1 -o gpurun_out/prof_gemm_s $CMD > gpurun_out/ncu_gemm.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_gemm.log
