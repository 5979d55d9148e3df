cd /root/repo
export SPCHOL_LIB=$PWD/paper_2409_14009_b200/libspchol.so
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name regex:"solve|permute" -c 3000 --csv --log-file gpurun_out/solve_launches_${CFG:-C2}.csv python scripts/solve_bench.py --config ${CFG:-C2} --reps 1 > gpurun_out/solve_ncu.log 2>&1
tail -3 gpurun_out/solve_ncu.log
