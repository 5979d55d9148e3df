#!/bin/bash
# Round-2 (second session) measurements on one B200: GPU test suite, smoke, C1-C5 bench lines, ncu launch
# lists (C4, C3), SYRK+scatter DRAM traffic of every launch (C4), --set full of the fused-cdiv kernels
# (C3 root), potrf10 and the largest SYRK+scatter launch, per-level wall times.  ncu numbers are never
# bench values.
set -u
mkdir -p gpurun_out
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > $O/r02b_gputest.log 2>&1; echo "rc=$?" >> $O/r02b_gputest.log
timeout 600 python __graft_entry__.py smoke > $O/r02b_smoke.log 2>&1; echo "rc=$?" >> $O/r02b_smoke.log
for C in C4 C1 C2 C3 C5; do
  timeout 900 python bench.py --config $C > $O/r02b_bench_$C.json 2> $O/r02b_bench_$C.err
done
timeout 900 python bench.py --impl reference > $O/r02b_reference_arm.json 2> $O/r02b_reference_arm.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv --log-file $O/r02b_launches_C4.csv \
    python scripts/one_factor.py C4 > $O/ncu_launch.log 2>&1
python scripts/summarize_launches.py $O/r02b_launches_C4.csv > $O/r02b_launches_C4_summary.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv --log-file $O/r02b_launches_C3.csv \
    python scripts/one_factor.py C3 > $O/ncu_launch3.log 2>&1
python scripts/summarize_launches.py $O/r02b_launches_C3.csv > $O/r02b_launches_C3_summary.txt 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active \
    --clock-control none --kernel-name-base demangled -k regex:'gemm_kernel<.int.2>' -c 200 --csv --log-file $O/r02b_scatter_dram_C4.csv \
    python scripts/one_factor.py C4 > $O/ncu_scatter.log 2>&1
ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:'gemm_kernel<.int.2>' --launch-skip 40 -c 1 \
    -o $O/r02b_scatter_full python scripts/one_factor.py C4 > $O/ncu_full.log 2>&1
ncu -i $O/r02b_scatter_full.ncu-rep --page details > $O/r02b_scatter_full_details.txt 2>/dev/null
ncu --set full --import-source on --clock-control none -k regex:panel_diag_kernel --launch-skip 60 -c 1 -o $O/r02b_panel_diag_full \
    python scripts/one_factor.py C3 > $O/ncu_pdiag.log 2>&1
ncu -i $O/r02b_panel_diag_full.ncu-rep --page details > $O/r02b_panel_diag_full_details.txt 2>/dev/null
ncu --set full --import-source on --clock-control none -k regex:panel_below_kernel --launch-skip 60 -c 1 -o $O/r02b_panel_below_full \
    python scripts/one_factor.py C3 > $O/ncu_pbelow.log 2>&1
ncu -i $O/r02b_panel_below_full.ncu-rep --page details > $O/r02b_panel_below_full_details.txt 2>/dev/null
ncu --set full --import-source on --clock-control none -k regex:potrf10_kernel --launch-skip 300 -c 1 -o $O/r02b_potrf10_full \
    python scripts/one_factor.py C4 > $O/ncu_potrf.log 2>&1
ncu -i $O/r02b_potrf10_full.ncu-rep --page details > $O/r02b_potrf10_full_details.txt 2>/dev/null
rm -f $O/*.ncu-rep
timeout 900 python scripts/level_profile.py C2 C3 C4 > $O/r02b_level_profile.txt 2>&1
timeout 300 python scripts/chain_bench.py 2048 4096 8192 15000 > $O/r02b_chain_bench.txt 2>&1
./tools/panel_probe 2048 > $O/r02b_panel_probe.txt 2>&1
