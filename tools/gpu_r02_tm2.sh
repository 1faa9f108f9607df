#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "tmem_sweep or ragged or c5" > gpurun_out/t_tm.log 2>&1; echo "tm tests rc=$?"; tail -5 gpurun_out/t_tm.log
timeout 300 python bench.py --no-cpu --no-e2e --no-tf32 --steps 20 --warmup 5 > gpurun_out/bench_tm.json 2> gpurun_out/bench_tm.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_tm.err
python -c "
import json
d=json.loads(open('gpurun_out/bench_tm.json').read().strip().splitlines()[-1])
p=d['roofline']['phases_ms']; print('it/s %.2f frac %.3f'%(d['value'], d['roofline']['frac']), d['sweeps'], {k: round(v,3) for k,v in p.items()})"
bash tools/gpu_sweep_prof.sh > /dev/null
grep "sweep_tm prof" gpurun_out/prof_run.json | awk '$8 == 10' | sort -k6,6n | awk 'NR%6==1' | head -8
