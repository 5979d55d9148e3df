#!/bin/bash
# below-launch grid cap sweep (SPCHOL_PANEL_GRID) with the fused cdiv on levels <= 16 large supernodes
set -u
mkdir -p gpurun_out
./tools/dmma_probe > gpurun_out/dmma_probe.txt 2>&1
for C in ${CONFIGS:-C3 C4}; do
  for G in ${SWEEP:-74 148 296}; do
    SPCHOL_PANEL_MAX_SN=${NSN:-16} SPCHOL_PANEL_GRID=$G timeout 600 python bench.py --config $C --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/pgrid_${C}_$G.json 2> gpurun_out/pgrid_${C}_$G.err
    echo "$C G=$G $(python -c "import json;d=json.loads(open('gpurun_out/pgrid_${C}_$G.json').read().strip().splitlines()[-1]);print(d['ms_per_step'])")" >> gpurun_out/pgrid.txt
  done
done
