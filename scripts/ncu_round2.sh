#!/bin/bash
# Round-2 ncu evidence (run under gpurun, one GPU): launch list of one C4 factor, DRAM traffic of every
# SYRK+scatter launch, --set full of the largest SYRK+scatter launch and of one POTRF.  Never a bench
# number (ncu serializes and replays).
set -u
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/r02_launches_C4.csv \
    python scripts/one_factor.py C4 > gpurun_out/ncu_launch.log 2>&1
python scripts/summarize_launches.py gpurun_out/r02_launches_C4.csv > gpurun_out/r02_launches_C4_summary.txt 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active \
    --clock-control none --kernel-name-base demangled -k regex:'gemm_kernel<.int.2>' -c 200 --csv --log-file gpurun_out/r02_scatter_dram_C4.csv \
    python scripts/one_factor.py C4 > gpurun_out/ncu_scatter.log 2>&1
ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:'gemm_kernel<.int.2>' --launch-skip 40 -c 1 \
    -o gpurun_out/r02_scatter_full python scripts/one_factor.py C4 > gpurun_out/ncu_full.log 2>&1
ncu -i gpurun_out/r02_scatter_full.ncu-rep --page details > gpurun_out/r02_scatter_full_details.txt 2>/dev/null
ncu --set full --clock-control none -k regex:potrf9 --launch-skip 200 -c 1 -o gpurun_out/r02_potrf9_full \
    python scripts/one_factor.py C3 > gpurun_out/ncu_potrf.log 2>&1
ncu -i gpurun_out/r02_potrf9_full.ncu-rep --page details > gpurun_out/r02_potrf9_full_details.txt 2>/dev/null
rm -f gpurun_out/*.ncu-rep
