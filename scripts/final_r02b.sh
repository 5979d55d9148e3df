#!/bin/bash
# End-of-round check on the final source: full -m gpu suite, smoke, the default bench line.
set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02c_gputest.log 2>&1; echo "rc=$?" >> gpurun_out/r02c_gputest.log
timeout 600 python __graft_entry__.py smoke > gpurun_out/r02c_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r02c_smoke.log
timeout 900 python bench.py > gpurun_out/r02c_bench_C4.json 2> gpurun_out/r02c_bench_C4.err
