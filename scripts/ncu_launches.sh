set -x
CFG=${CFG:-C4}
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${CFG}.csv python scripts/profile_factor.py --config $CFG > gpurun_out/ncu_launch.log 2>&1
tail -3 gpurun_out/ncu_launch.log
ncu --set full --clock-control none --import-source on -k regex:potrf -s 20 -c 2 -o gpurun_out/prof_potrf python scripts/profile_factor.py --config $CFG > gpurun_out/ncu_full1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 300 -c 6 -o gpurun_out/prof_gemm python scripts/profile_factor.py --config $CFG > gpurun_out/ncu_full2.log 2>&1
tail -3 gpurun_out/ncu_full2.log
ls -la gpurun_out
