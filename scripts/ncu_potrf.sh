ncu --section SourceCounters --section WarpStateStats --section LaunchStats --section SpeedOfLight --warp-sampling-interval 0 --clock-control none --import-source on -k regex:potrf -s 480 -c 1 -o gpurun_out/prof_potrf8 python scripts/profile_factor.py --config C4 > gpurun_out/ncu_full1.log 2>&1
tail -1 gpurun_out/ncu_full1.log
