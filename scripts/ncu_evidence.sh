# 1) launch list of one C4 factor (device time per launch, cold-cache and serialized)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches_C4.csv python scripts/profile_factor.py --config C4 > /dev/null 2>&1
# 2) DRAM traffic of every SYRK+scatter launch (dominant kernel) in one C4 factor
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --kernel-name-base mangled -k regex:gemm_kernelILi2 --csv --log-file gpurun_out/r01_scatter_dram_C4.csv python scripts/profile_factor.py --config C4 > /dev/null 2>&1
# 3) full set on the largest scatter launches and a large in-panel update launch
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:gemm_kernelILi2 -s 9 -c 1 -o gpurun_out/r01_scatter_full python scripts/profile_factor.py --config C4 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:gemm_kernelILi0 -s 1200 -c 1 -o gpurun_out/r01_local_full python scripts/profile_factor.py --config C4 > /dev/null 2>&1
ls -la gpurun_out | tail
