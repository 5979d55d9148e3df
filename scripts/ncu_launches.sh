CFG=${CFG:-C4}
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${CFG}.csv python scripts/profile_factor.py --config $CFG > gpurun_out/ncu_launch.log 2>&1
tail -1 gpurun_out/ncu_launch.log
