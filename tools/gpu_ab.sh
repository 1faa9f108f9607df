#!/bin/bash
# A/B of HALS sweep variants + tests.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for v in ${VARIANTS:-default p12 dmma1}; do
  ENMF_HALS_KERNEL=$v python bench.py --no-cpu --no-e2e --steps 10 > gpurun_out/bench_$v.json 2> gpurun_out/bench_$v.err
done
