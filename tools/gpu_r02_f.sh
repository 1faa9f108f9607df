timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "tf32" > gpurun_out/t_tf32.log 2>&1; echo "tf32 rc=$?"; tail -3 gpurun_out/t_tf32.log
timeout 300 python bench.py --no-cpu --no-e2e --steps 5 --warmup 3 > gpurun_out/bench_f.json 2> gpurun_out/bench_f.err; echo "bench rc=$?"; tail -2 gpurun_out/bench_f.err
python -c "
import json
d=json.loads(open('gpurun_out/bench_f.json').read().strip().splitlines()[-1])
print('fp64 it/s %.2f'%d['value']); print('tf32', json.dumps(d.get('tf32_variant'))[:600])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tf32k" -c 6 --csv python bench.py --no-cpu --no-e2e --steps 1 --warmup 1 2>/dev/null | grep tf32k | cut -c1-60,200-
