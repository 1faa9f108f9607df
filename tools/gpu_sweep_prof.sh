#!/bin/bash
# clock64 phase profile of sweep_tm (libenmf_gpu_prof.so, -DENMF_SWEEP_PROF): cycles per sweep by phase
mkdir -p gpurun_out
ENMF_GPU_LIB=$PWD/paper_1805_06604_b200/libenmf_gpu_prof.so timeout 300 python bench.py --no-cpu --no-e2e --no-tf32 --steps 3 --warmup 3 > gpurun_out/prof_run.json 2> gpurun_out/prof_run.err
grep "sweep_tm prof" gpurun_out/prof_run.json gpurun_out/prof_run.err | awk '$8 > 100' | tail -16
