#!/bin/bash
# compute-sanitizer over the fused outer-block cdiv (panel_diag_kernel / panel_below_kernel, potrf10
# inside and standalone), forced on every level and outer block.  Logs: gpurun_out/r02b_sanitizer_panel_*.log
set -u
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
export SPCHOL_PANEL_MAX_SN=1000000 SPCHOL_PANEL_MAX_ROWS=1000000000
for tool in memcheck racecheck synccheck initcheck; do
  for cfg in "T3 -1" "S4 -1" "S5 -1" "C1 -1"; do
    set -- $cfg
    echo "=== $tool $cfg (fused path forced)" >> gpurun_out/r02b_sanitizer_panel_$tool.log
    timeout 1200 $CS --tool $tool --error-exitcode 9 python scripts/sanitize_run.py $1 $2 >> gpurun_out/r02b_sanitizer_panel_$tool.log 2>&1
    echo "exit $?" >> gpurun_out/r02b_sanitizer_panel_$tool.log
  done
done
