CFG=${CFG:-C4}
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
ncu --set full --clock-control none --import-source on -k regex:potrf -s 400 -c 2 -o gpurun_out/prof_potrf3 python scripts/profile_factor.py --config $CFG > gpurun_out/ncu_full1.log 2>&1
tail -2 gpurun_out/ncu_full1.log
