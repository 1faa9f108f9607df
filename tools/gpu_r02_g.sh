timeout 900 python -m pytest tests/test_gpu_boundary.py tests/test_gpu_parity.py -q -x -k "boundary or namespace or non_finite or bpp_wide or wide_rank" > gpurun_out/t_g1.log 2>&1; echo "new tests rc=$?"; tail -15 gpurun_out/t_g1.log
timeout 2000 python -m pytest tests/test_gpu_sanitize.py -q > gpurun_out/t_san.log 2>&1; echo "sanitize rc=$?"; tail -30 gpurun_out/t_san.log
