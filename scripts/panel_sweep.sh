#!/bin/bash
# SPCHOL_PANEL_MAX_SN sweep (fused cdiv only in levels with <= N large supernodes; 0 = never)
set -u
mkdir -p gpurun_out
for C in ${CONFIGS:-C2 C3 C4}; do
  for N in ${SWEEP:-0 2 4 8 16}; do
    SPCHOL_PANEL_MAX_SN=$N timeout 600 python bench.py --config $C --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/psweep_${C}_$N.json 2> gpurun_out/psweep_${C}_$N.err
    echo "$C N=$N $(python -c "import json;d=json.loads(open('gpurun_out/psweep_${C}_$N.json').read().strip().splitlines()[-1]);print(d['ms_per_step'])")" >> gpurun_out/psweep.txt
  done
done
