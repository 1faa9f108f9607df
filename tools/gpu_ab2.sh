#!/bin/bash
# Parity tests (default kernels) + A/B of HALS sweep variants at the default step count.
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for v in ${VARIANTS:-ws t14u2}; do
  ENMF_HALS_KERNEL=$v timeout 300 python bench.py --no-cpu --no-e2e ${BENCH_ARGS:-} > gpurun_out/bench_$v.json 2> gpurun_out/bench_$v.err
done
