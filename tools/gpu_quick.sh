#!/bin/bash
# Quick GPU iteration: tests + bench (both HALS kernels) without ncu.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python bench.py --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
ENMF_HALS_KERNEL=fma python bench.py --no-cpu --no-e2e --steps 10 > gpurun_out/bench_fma.json 2> gpurun_out/bench_fma.err
