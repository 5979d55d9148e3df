export SPCHOL_LIB=$PWD/paper_2409_14009_b200/libspchol.so
python -m pytest tests/ -m gpu -x -q 2>&1 | tail -1
for c in ${CFGS:-C2 C4}; do python scripts/variant_bench.py --config $c | grep lib | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config'], round(d['ms'],2), {k:v['ms'] for k,v in d['kernels'].items()})"; done
