timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "gpu tests rc=$?"; tail -15 gpurun_out/pytest_gpu.log
