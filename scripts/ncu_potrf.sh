ncu --set full --clock-control none --import-source on -k regex:potrf -s 480 -c 3 -o gpurun_out/prof_potrf7 python scripts/profile_factor.py --config C4 > gpurun_out/ncu_full1.log 2>&1
tail -1 gpurun_out/ncu_full1.log
