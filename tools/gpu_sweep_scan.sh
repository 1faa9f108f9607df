#!/bin/bash
# device time of one persistent sweep_tm launch per solve length (ncu gpu__time_duration), for the
# in-tree build and $PREV
mkdir -p gpurun_out
for lib in "" $PREV; do
  ENMF_GPU_LIB=$lib timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"sweep_tm|sweep_ws" --csv python tools/sweep_scan.py 2>/dev/null | grep -E "sweep_(tm|ws)" | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' '
  echo " <- ${lib:-current} (ns per launch for sweeps 2 4 8 16 32 64 129 129 64 8)"
done
