./tools/probe/umma_rate_probe > gpurun_out/umma_rate.txt 2>&1; cat gpurun_out/umma_rate.txt
for v in ss ts2; do
ENMF_OZK=$v timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,lts__t_sectors.sum.pct_of_peak_sustained_elapsed,dram__bytes_read.sum.pct_of_peak_sustained_elapsed,l1tex__m_xbar2l1tex_read_bytes.sum.per_second --clock-control none -k regex:gemm_levels -s 2 -c 1 python bench.py --no-cpu --no-e2e --no-tf32 --steps 1 --warmup 1 > gpurun_out/ncu_m_$v.txt 2>&1
grep -E "gemm_levels|duration|pct|second" gpurun_out/ncu_m_$v.txt | head -12
done
