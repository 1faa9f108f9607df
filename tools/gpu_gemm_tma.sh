#!/bin/bash
# TMA-fed FP64 DMMA GEMM (gemm_f64_dmma_t) vs the cp.async loader (gemm_f64_dmma_s): parity + A/B.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for L in tma cpasync; do
  ENMF_GEMM_LOAD=$L timeout 600 python bench.py --warmup 5 --no-cpu > gpurun_out/bench_$L.json 2> gpurun_out/bench_$L.err
  for w in c2 c3 c4; do
    ENMF_GEMM_LOAD=$L timeout 600 python bench.py --workload $w --steps 300 --warmup 5 --no-cpu --no-e2e > gpurun_out/bench_${w}_$L.json 2> gpurun_out/bench_${w}_$L.err
  done
done
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_f64_dmma_t -s 4 -c 1 -o gpurun_out/prof_gemmt -f $CMD > gpurun_out/ncu_gemmt.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --workload c2 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_c2.log 2>&1
ENMF_GEMM_LOAD=cpasync timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_cp.csv python bench.py --workload c2 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_c2cp.log 2>&1
[ -f gpurun_out/prof_gemmt.ncu-rep ] && python tools/ncu_report.py gpurun_out/prof_gemmt.ncu-rep gemmt > gpurun_out/summary_gemmt.txt 2>&1
rm -f gpurun_out/prof_gemmt.ncu-rep
