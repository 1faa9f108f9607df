#!/bin/bash
# ncu --set full of one sweep_tm launch (8 sweeps at C5 size via enmf_gpu_hals_solve), current build
# and $PREV (an earlier build of libenmf_gpu.so) for comparison
mkdir -p gpurun_out
export SWEEP_LONG=16
timeout 600 ncu --set full --import-source on --clock-control none -k regex:sweep_tm -s 2 -c 1 -o gpurun_out/prof_tm -f python tools/sweep_bench.py > gpurun_out/ncu_tm.log 2>&1; echo "ncu rc=$?"
if [ -n "$PREV" ]; then
ENMF_GPU_LIB=$PREV timeout 600 ncu --set full --import-source on --clock-control none -k regex:sweep_tm -s 2 -c 1 -o gpurun_out/prof_tm_prev -f python tools/sweep_bench.py > gpurun_out/ncu_tm_prev.log 2>&1; echo "ncu prev rc=$?"
fi
python tools/sweep_bench.py 2>&1 | tail -1
ENMF_GPU_LIB=$PREV python tools/sweep_bench.py 2>&1 | tail -1
