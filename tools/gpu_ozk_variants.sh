# A/B of the digit-GEMM variants (ENMF_OZK): parity subset + C5 cross-product time per variant
for v in ${VARIANTS:-ss ts ts2 ss2 ts4}; do
  ENMF_OZK=$v timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "int8 or ragged" > gpurun_out/t_ozk_$v.log 2>&1
  echo "$v parity rc=$? $(tail -1 gpurun_out/t_ozk_$v.log)"
  ENMF_OZK=$v timeout 200 python bench.py --no-cpu --no-e2e --no-tf32 --steps 5 --warmup 3 > gpurun_out/b_ozk_$v.json 2> gpurun_out/b_ozk_$v.err
  python -c "
import json,sys
d=json.loads(open('gpurun_out/b_ozk_$v.json').read().strip().splitlines()[-1])
p=d['roofline']['phases_ms']; print('$v', 'it/s %.2f'%d['value'], 'cross_wx %.3f cross_xht %.3f'%(p['cross_wx'],p['cross_xht']))" || tail -3 gpurun_out/b_ozk_$v.err
done
