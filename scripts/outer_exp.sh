export SPCHOL_LIB=$PWD/paper_2409_14009_b200/libspchol.so
for o in 2 4 6 8; do for c in C4 C3; do SPCHOL_OUTER=$o timeout 200 python scripts/variant_bench.py --config $c | grep lib | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('outer', $o, d['config'], round(d['ms'],2), {k:v['ms'] for k,v in d['kernels'].items()})"; done; done
SPCHOL_OUTER=8 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "configs or block" 2>&1 | tail -1
