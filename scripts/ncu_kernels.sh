# --set full captures of the non-dominant kernels of one C4 factor (profiles/r01_kernels_C4.txt)
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:potrf8 -s 900 -c 1 -o gpurun_out/k_potrf python scripts/profile_factor.py --config C4 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:gemm_kernelILi0 -s 1300 -c 1 -o gpurun_out/k_local python scripts/profile_factor.py --config C4 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:gemm_kernelILi1 -s 900 -c 1 -o gpurun_out/k_trsm python scripts/profile_factor.py --config C4 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:small_warp_kernel -s 3 -c 1 -o gpurun_out/k_smallw python scripts/profile_factor.py --config C2 > /dev/null 2>&1
ls gpurun_out/k_*
