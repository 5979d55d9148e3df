#!/bin/bash
# ncu --set full of one potrf8_kernel launch (dense 2048 chain) with source-level counters.
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none --warp-sampling-interval 0 -k regex:potrf8 -s 5 -c 1 -o gpurun_out/potrf8 \
    python scripts/chain_bench.py 2048 > gpurun_out/ncu_potrf.log 2>&1
ncu -i gpurun_out/potrf8.ncu-rep --page source --csv > gpurun_out/potrf8_source.csv 2>/dev/null
ncu -i gpurun_out/potrf8.ncu-rep --page raw --csv > gpurun_out/potrf8_raw.csv 2>/dev/null
ncu -i gpurun_out/potrf8.ncu-rep --page details > gpurun_out/potrf8_details.txt 2>/dev/null
