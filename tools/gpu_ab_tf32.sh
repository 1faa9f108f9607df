mkdir -p gpurun_out
for rep in 1 2; do
  ENMF_GPU_LIB=/root/repo/libenmf_gpu_base.so timeout 600 python bench.py --no-cpu --no-e2e --steps 20 > gpurun_out/bench_base$rep.json 2>/dev/null
  timeout 600 python bench.py --no-cpu --no-e2e --steps 20 > gpurun_out/bench_new$rep.json 2>/dev/null
done
timeout 900 python -m pytest tests -m gpu -x -q -k "tf32" > gpurun_out/pytest.log 2>&1
