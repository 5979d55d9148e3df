# DRAM traffic, L2 hit rate, DMMA utilisation and grid size of every in-panel update launch (gemm_kernel<0>) of one C4 factor
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct,launch__grid_size --clock-control none --kernel-name-base mangled -k regex:gemm_kernelILi0 --csv --log-file gpurun_out/local_dram_C4.csv python scripts/profile_factor.py --config C4 > gpurun_out/ncu_local.log 2>&1
tail -3 gpurun_out/ncu_local.log
wc -l gpurun_out/local_dram_C4.csv
