set -x
timeout 900 python -m pytest tests/ -m gpu -q 2>&1 | tail -1
for c in C1 C2 C3 C5; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/bench_$c.json; done
timeout 600 python bench.py --steps 5 --warmup 3 2>/dev/null | tail -1 > gpurun_out/bench_C4.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C4.csv python scripts/profile_factor.py --config C4 > /dev/null 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --kernel-name-base mangled -k regex:gemm_kernelILi2 --csv --log-file gpurun_out/scatter_dram_C4.csv python scripts/profile_factor.py --config C4 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:gemm_kernelILi2 -s 40 -c 1 -o gpurun_out/scatter_full python scripts/profile_factor.py --config C4 > /dev/null 2>&1
ls gpurun_out
