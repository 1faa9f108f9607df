set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "int8 or ragged or sharded or eanls_large" > gpurun_out/t_int8.log 2>&1; echo "int8 rc=$?"
tail -5 gpurun_out/t_int8.log
timeout 300 python bench.py --no-cpu --no-e2e --no-tf32 --steps 10 --warmup 3 > gpurun_out/bench_tc.json 2> gpurun_out/bench_tc.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench_tc.json; tail -5 gpurun_out/bench_tc.err
timeout 1200 python -m pytest tests/test_gpu_long.py -q -x > gpurun_out/t_long.log 2>&1; echo "long rc=$?"
tail -15 gpurun_out/t_long.log
