export SPCHOL_LIB=$PWD/paper_2409_14009_b200/libspchol.so
timeout 600 python -m pytest tests/ -m gpu -x -q 2>&1 | grep -E "passed|failed|^E " | head -3; echo
for c in C4 C3 C2; do timeout 200 python scripts/variant_bench.py --config $c | grep lib | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config'], round(d['ms'],2))"; done
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:potrf -s 480 -c 5 --csv python scripts/profile_factor.py --config C4 2>/dev/null | grep -o '"[0-9.]*"$' | tr '\n' ' '; echo
