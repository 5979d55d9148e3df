export SPCHOL_LIB=$PWD/paper_2409_14009_b200/libspchol.so
for L in $LEVELS; do SPCHOL_MAX_LEVEL=$L python scripts/variant_bench.py --config $CFG | grep lib | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($L, round(d['ms'],3))"; done
