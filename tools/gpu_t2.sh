#!/bin/bash
# A/B of the two-team HALS sweep (ENMF_HALS_KERNEL=t2) against the default paired-warp sweep.
mkdir -p gpurun_out
VARIANTS="wsp t2" bash tools/sweep_breakdown.sh
ENMF_HALS_KERNEL=t2 timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_t2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_t2.log
ENMF_HALS_KERNEL=t2 timeout 600 python bench.py --no-cpu --no-e2e --steps 10 > gpurun_out/bench_t2.json 2> gpurun_out/bench_t2.err
timeout 600 python bench.py --no-cpu --no-e2e --steps 10 > gpurun_out/bench_wsp.json 2> gpurun_out/bench_wsp.err
