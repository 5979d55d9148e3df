ncu --set full --clock-control none --import-source on -k regex:small_kernel -s 1 -c 1 -o gpurun_out/prof_small python scripts/profile_factor.py --config C2 > gpurun_out/ncu_small.log 2>&1
tail -1 gpurun_out/ncu_small.log
