# the driver's bench commands: our arm, then the reference arm (same window)
nproc; free -g | head -2
( time python bench.py --steps ${K:-20} --warmup ${W:-5} > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err ) 2>&1 | tail -3
tail -c 400 gpurun_out/bench_full.err
( time python bench.py --impl reference --steps ${K:-20} --warmup ${W:-5} > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err ) 2>&1 | tail -3
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_full.json').read().strip().splitlines()[-1])
r=json.loads(open('gpurun_out/bench_ref.json').read().strip().splitlines()[-1])
print('ours', round(d['value'],2), 'e2e', d['e2e'] and round(d['e2e']['value'],2), 'roof', round(d['roofline']['frac'],3), 'cpu', d['cpu_baseline'] and d['cpu_baseline'].get('value'))
print('tf32', d['tf32_variant'] and {k: d['tf32_variant'][k] for k in ('value','abs_diff','within_1e-4')})
print('ref', r['value'], r['sweeps'])
print('ratio', d['value']/r['value'], 'e2e ratio', d['e2e']['value']/r['value'] if d['e2e'] else None)
print('phases', {k: round(v,3) for k,v in d['roofline']['phases_ms'].items()})
print('sweeps', d['sweeps'], 'clocks', d['clocks'])
PY
