#!/bin/bash
# A/B of the fused outer-block cdiv (SPCHOL_PANEL=1, default) against separate POTRF/TRSM/update
# launches (SPCHOL_PANEL=0): parity subset, dense chain benchmark, C2/C3/C4 factor times.
set -u
mkdir -p gpurun_out
rm -f gpurun_out/panel_chain.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "${PARITY_K:-parity_configs or block_sizes or not_spd or edge or random_corpus or schedule_options or distributed_nccl or memory_capped_parity}" > gpurun_out/panel_parity.log 2>&1
echo "parity rc=$?" >> gpurun_out/panel_parity.log
for P in 1 0; do
  echo "== PANEL=$P" >> gpurun_out/panel_chain.txt
  SPCHOL_PANEL=$P timeout 300 python scripts/chain_bench.py 2048 4096 8192 >> gpurun_out/panel_chain.txt 2>&1
done
for C in ${CONFIGS:-C2 C3 C4}; do
  for P in 1 0; do
    SPCHOL_PANEL=$P timeout 600 python bench.py --config $C --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/panel_${C}_$P.json 2> gpurun_out/panel_${C}_$P.err
  done
done
