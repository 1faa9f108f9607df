#!/bin/bash
# One GPU call: tests, smoke, bench, ncu launch list + full captures of the dominant kernels.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
if [ "${NCU:-1}" = "1" ]; then
  CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
  timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_ws -s 2 -c 1 -o gpurun_out/prof_sweep $CMD > gpurun_out/ncu_sweep.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"i256x256x32gemm_s8" -s 6 -c 6 -o gpurun_out/prof_i8 $CMD > gpurun_out/ncu_i8.log 2>&1
  echo "ncu rc=$?" >> gpurun_out/ncu_i8.log
fi
