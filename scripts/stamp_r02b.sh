#!/bin/bash
# Final stamp of round 2: DRAM traffic of every SYRK+scatter launch of one C4 factor on the committed
# kernel source (profiles/roofline_traffic.json is regenerated from it), then the default bench line.
set -u
mkdir -p gpurun_out
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active \
    --clock-control none --kernel-name-base demangled -k regex:'gemm_kernel<.int.2>' -c 200 --csv --log-file gpurun_out/r02c_scatter_dram_C4.csv \
    python scripts/one_factor.py C4 > gpurun_out/ncu_scatter.log 2>&1
python scripts/make_traffic_json.py gpurun_out/r02c_scatter_dram_C4.csv > gpurun_out/make_traffic.log 2>&1
cp profiles/roofline_traffic.json gpurun_out/roofline_traffic.json
timeout 900 python bench.py > gpurun_out/r02c_bench_C4.json 2> gpurun_out/r02c_bench_C4.err
