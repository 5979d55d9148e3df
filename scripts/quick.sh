export SPCHOL_LIB=$PWD/paper_2409_14009_b200/libspchol.so
timeout 600 python -m pytest tests/ -m gpu -x -q 2>&1 | grep -E "passed|failed"
for c in ${CFGS:-C2 C4}; do timeout 200 python scripts/variant_bench.py --config $c | grep lib | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config'], round(d['ms'],2), {k:v['ms'] for k,v in d['kernels'].items()})"; done
