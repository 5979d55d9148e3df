#!/bin/bash
# SPCHOL_PANEL_MAX_ROWS sweep (fused cdiv for outer blocks with m - c0 <= R rows, chain-critical levels)
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "parity_configs or block_sizes or not_spd or edge or random_corpus or schedule_options or distributed_nccl or memory_capped_parity" > gpurun_out/panel_parity.log 2>&1
echo "parity rc=$?" >> gpurun_out/panel_parity.log
for C in ${CONFIGS:-C2 C3 C4}; do
  for R in ${SWEEP:-0 4096 8192 16384}; do
    SPCHOL_PANEL_MAX_ROWS=$R timeout 600 python bench.py --config $C --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prows_${C}_$R.json 2> gpurun_out/prows_${C}_$R.err
    echo "$C R=$R $(python -c "import json;d=json.loads(open('gpurun_out/prows_${C}_$R.json').read().strip().splitlines()[-1]);print(d['ms_per_step'])")" >> gpurun_out/prows.txt
  done
done
