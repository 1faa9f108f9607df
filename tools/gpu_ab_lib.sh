#!/bin/bash
# Same-box A/B of two builds of libenmf_gpu.so: $AB_BASE (ENMF_GPU_LIB) against the in-tree build.
mkdir -p gpurun_out
for rep in 1 2; do
  ENMF_GPU_LIB=$AB_BASE timeout 600 python bench.py --no-cpu --no-e2e --steps 20 > gpurun_out/bench_base$rep.json 2>/dev/null
  timeout 600 python bench.py --no-cpu --no-e2e --steps 20 > gpurun_out/bench_new$rep.json 2>/dev/null
done
