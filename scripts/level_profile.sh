# Cumulative factor time with levels <= L (SPCHOL_MAX_LEVEL) and the serialized per-level kernel times.
CFG=${CFG:-C4}
python scripts/variant_bench.py --config $CFG --steps 3 > gpurun_out/level_full_$CFG.json
for L in $LEVELS; do SPCHOL_MAX_LEVEL=$L python scripts/variant_bench.py --config $CFG --steps 3 | grep lib | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($L, round(d['ms'],3))"; done > gpurun_out/level_cum_$CFG.txt
cat gpurun_out/level_cum_$CFG.txt
