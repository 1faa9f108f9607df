set -x
timeout 1500 python -m pytest tests/test_gpu_long.py -q -x -s > gpurun_out/t_long.log 2>&1; echo "long rc=$?"
tail -15 gpurun_out/t_long.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm_levels|finish|split_rows|row_absmax|sweep_ws" -c 40 --csv python bench.py --no-cpu --no-e2e --no-tf32 --steps 1 --warmup 1 > gpurun_out/ncu_tc_launch.csv 2> gpurun_out/ncu_tc_launch.err; echo "ncu1 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_levels -s 2 -c 1 -o gpurun_out/prof_tc python bench.py --no-cpu --no-e2e --no-tf32 --steps 1 --warmup 1 > gpurun_out/ncu_tc.log 2>&1; echo "ncu2 rc=$?"
tail -3 gpurun_out/ncu_tc.log
