export SPCHOL_LIB=$PWD/paper_2409_14009_b200/libspchol.so
python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
python scripts/variant_bench.py | grep lib | cut -c1-300
python scripts/variant_bench.py --config C3 | grep lib | cut -c1-120
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:potrf -s 480 -c 5 --csv python scripts/profile_factor.py --config C4 2>/dev/null | grep -o '"[0-9.]*"$' | tr '\n' ' '; echo
