ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:gemm_tma_kernelILi2 -s 9 -c 1 -o gpurun_out/prof_tma python scripts/profile_factor.py --config C4 > gpurun_out/ncu_tma.log 2>&1
tail -1 gpurun_out/ncu_tma.log
