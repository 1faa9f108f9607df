# launch list of the cross-product kernels + one full ncu capture of the digit GEMM
V=${V:-c2}
ENMF_OZK=$V timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm_levels|finish|split_rows|row_absmax" -c 12 --csv python bench.py --no-cpu --no-e2e --no-tf32 --steps 1 --warmup 1 > gpurun_out/ncu_launch_$V.csv 2> /dev/null
ENMF_OZK=$V timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_levels -s 2 -c 1 -o gpurun_out/prof_ozk_$V python bench.py --no-cpu --no-e2e --no-tf32 --steps 1 --warmup 1 > gpurun_out/ncu_ozk_$V.log 2>&1; echo "ncu rc=$?"
