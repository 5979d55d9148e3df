export SPCHOL_LIB=$PWD/paper_2409_14009_b200/libspchol.so
timeout 600 python -m pytest tests/ -m gpu -x -q 2>&1 | grep -E "passed|failed|^E " | head -5
for c in C2 C3 C4; do for vr in 1 2 4 8; do timeout 200 python scripts/variant_bench.py --config $c --vr $vr | grep lib | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config'], 'vr', d['vr'], round(d['ms'],2))"; done; done
