timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-cpu --no-e2e --no-tf32 --steps 10 --warmup 5 > gpurun_out/bench_e.json 2> gpurun_out/bench_e.err
python -c "
import json
d=json.loads(open('gpurun_out/bench_e.json').read().strip().splitlines()[-1])
p=d['roofline']['phases_ms']; print('it/s %.2f'%d['value'], {k: round(v,3) for k,v in p.items()})"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"finish" -c 4 --csv python bench.py --no-cpu --no-e2e --no-tf32 --steps 1 --warmup 1 2>/dev/null | grep finish | head -4
