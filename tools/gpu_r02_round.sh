#!/bin/bash
# Round-2 GPU call: tests, smoke, bench (+reference arm), launch list, ncu full captures of the
# dominant kernels (persistent sweep, tcgen05 digit GEMM, tcgen05 TF32 GEMM, DMMA Gram GEMM).
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt
if [ "${TESTS:-1}" = "1" ]; then
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
fi
timeout 900 python bench.py --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
if [ "${REF:-1}" = "1" ]; then
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
fi
if [ "${NCU:-1}" = "1" ]; then
  CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
  timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
  echo "launch rc=$?" >> gpurun_out/ncu_launch.log
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep_ws -s 2 -c 1 -o gpurun_out/prof_sweep -f $CMD > gpurun_out/ncu_sweep.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_levels -s 2 -c 1 -o gpurun_out/prof_ozk -f $CMD > gpurun_out/ncu_ozk.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"ozk::finish|finish<" -s 2 -c 1 -o gpurun_out/prof_finish -f $CMD > gpurun_out/ncu_finish.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"tf32k::gemm|gemm\(tf32k" -s 2 -c 1 -o gpurun_out/prof_tf32k -f $CMD > gpurun_out/ncu_tf32k.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_f64_dmma_s -s 4 -c 1 -o gpurun_out/prof_gram -f $CMD > gpurun_out/ncu_gram.log 2>&1
  echo "ncu done" >> gpurun_out/ncu_gram.log
fi
