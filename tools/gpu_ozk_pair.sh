#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "int8 or ragged or c5 or wide_dynamic" > gpurun_out/t_pair.log 2>&1; echo "int8 tests rc=$?"; tail -4 gpurun_out/t_pair.log
for v in "" c2; do
ENMF_OZK=$v timeout 300 python bench.py --no-cpu --no-e2e --no-tf32 --steps 20 --warmup 5 > gpurun_out/bench_ozk$v.json 2> gpurun_out/bench_ozk$v.err; echo "bench $v rc=$?"; tail -2 gpurun_out/bench_ozk$v.err
python -c "
import json
d=json.loads(open('gpurun_out/bench_ozk$v.json').read().strip().splitlines()[-1])
p=d['roofline']['phases_ms']; print('ozk=$v it/s %.2f'%d['value'], 'cross', round(p['cross_wx'],3), round(p['cross_xht'],3), 'final', d.get('final_relative_error'))"
done
timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed --clock-control none -k regex:gemm_pair -s 2 -c 2 python bench.py --no-cpu --no-e2e --no-tf32 --steps 1 --warmup 1 2>/dev/null | grep -E "gemm_pair|duration|pct|bytes" | head -14
