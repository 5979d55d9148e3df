set -u
mkdir -p gpurun_out
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active \
    --clock-control none --kernel-name-base demangled -k regex:'gemm_kernel<.int.2>' -c 200 --csv --log-file gpurun_out/r02_scatter_dram_C4.csv \
    python scripts/one_factor.py C4 > gpurun_out/ncu_scatter.log 2>&1
ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:'gemm_kernel<.int.2>' --launch-skip 40 -c 1 \
    -o gpurun_out/r02_scatter_full python scripts/one_factor.py C4 > gpurun_out/ncu_full.log 2>&1
ncu -i gpurun_out/r02_scatter_full.ncu-rep --page details > gpurun_out/r02_scatter_full_details.txt 2>/dev/null
rm -f gpurun_out/*.ncu-rep
