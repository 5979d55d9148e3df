export SPCHOL_LIB=$PWD/paper_2409_14009_b200/libspchol.so
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | grep -E "passed|failed|Error|^E " | head -5
for c in C4 C3; do
SPCHOL_NO_TMA=1 python scripts/variant_bench.py --config $c | grep lib | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('notma', d['config'], round(d['ms'],2), {k:(v['ms'],v['tf']) for k,v in d['kernels'].items()})"
python scripts/variant_bench.py --config $c | grep lib | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tma  ', d['config'], round(d['ms'],2), {k:(v['ms'],v['tf']) for k,v in d['kernels'].items()})"
done
