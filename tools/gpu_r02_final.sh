#!/bin/bash
# Round-2 measurement call: tests, smoke, bench (+reference arm), launch list, ncu --set full
# captures of the kernels the profiles/ summaries cite.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt
if [ "${TESTS:-1}" = "1" ]; then
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
fi
timeout 900 python bench.py --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 python bench.py --workload c2 --steps 500 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python bench.py --workload c3 --steps 100 --warmup 5 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 python bench.py --workload c4 --steps 300 --warmup 5 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
if [ "${REF:-1}" = "1" ]; then
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
fi
python tools/batch_throughput.py > gpurun_out/batch_throughput.txt 2>&1
if [ "${NCU:-1}" = "1" ]; then
  CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
  timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
  echo "launch rc=$?" >> gpurun_out/ncu_launch.log
  SWEEP_LONG=16 timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep_tm -s 2 -c 1 -o gpurun_out/prof_tm -f python tools/sweep_bench.py > gpurun_out/ncu_tm.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_pair -s 2 -c 1 -o gpurun_out/prof_pair -f $CMD > gpurun_out/ncu_pair.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"ozk::finish" -s 2 -c 1 -o gpurun_out/prof_finish -f $CMD > gpurun_out/ncu_finish.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"tf32k::gemm" -s 2 -c 1 -o gpurun_out/prof_tf32k -f $CMD > gpurun_out/ncu_tf32k.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_f64_dmma_t -s 4 -c 1 -o gpurun_out/prof_gram -f $CMD > gpurun_out/ncu_gram.log 2>&1
  SWEEP_PREC=tf32 timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep_rl -s 6 -c 1 -o gpurun_out/prof_rl -f python tools/sweep_scan.py > gpurun_out/ncu_rl.log 2>&1
  BATCH=296 timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"batch::run" -s 1 -c 1 -o gpurun_out/prof_batch -f python tools/batch_throughput.py > gpurun_out/ncu_batch.log 2>&1
  echo "ncu done" >> gpurun_out/ncu_batch.log
  # summarise on the box, keep only the sweep capture (gpurun copies back <= 64 MiB)
  for f in tm pair finish tf32k gram batch rl; do
    [ -f gpurun_out/prof_$f.ncu-rep ] && python tools/ncu_report.py gpurun_out/prof_$f.ncu-rep "$f" > gpurun_out/summary_$f.txt 2>&1
  done
  rm -f gpurun_out/prof_pair.ncu-rep gpurun_out/prof_finish.ncu-rep gpurun_out/prof_tf32k.ncu-rep gpurun_out/prof_gram.ncu-rep gpurun_out/prof_batch.ncu-rep gpurun_out/prof_rl.ncu-rep
fi
