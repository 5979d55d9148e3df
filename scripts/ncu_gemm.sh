CFG=${CFG:-C4}
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:gemm_kernelILi2 -s 8 -c 2 -o gpurun_out/prof_scatter python scripts/profile_factor.py --config $CFG > gpurun_out/ncu_s.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:gemm_kernelILi0 -s 300 -c 3 -o gpurun_out/prof_local python scripts/profile_factor.py --config $CFG > gpurun_out/ncu_l.log 2>&1
tail -2 gpurun_out/ncu_s.log gpurun_out/ncu_l.log
