#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for v in 64 128; do
  ENMF_GEMM_TILE=$v python bench.py --no-cpu --no-e2e --steps 5 > gpurun_out/bench_t$v.json 2> gpurun_out/bench_t$v.err
done
