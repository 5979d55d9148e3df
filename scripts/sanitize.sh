#!/bin/bash
# compute-sanitizer over small configs: every tool, every kernel path (fused small kernels, tiled
# path with small_max_k=-1).  Logs go to gpurun_out/sanitizer_*.log.
set -u
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  for cfg in "T3 0" "T3 -1" "S4 -1" "C1 0"; do
    set -- $cfg
    echo "=== $tool $cfg" >> gpurun_out/sanitizer_$tool.log
    timeout 900 $CS --tool $tool --error-exitcode 9 python scripts/sanitize_run.py $1 $2 >> gpurun_out/sanitizer_$tool.log 2>&1
    echo "exit $?" >> gpurun_out/sanitizer_$tool.log
  done
done
