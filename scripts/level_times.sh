export SPCHOL_LIB=$PWD/paper_2409_14009_b200/libspchol.so
for L in 4 7 9 10 11 12; do SPCHOL_MAX_LEVEL=$L python scripts/variant_bench.py --config ${CFG:-C4} | grep lib | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($L, round(d['ms'],2))"; done
