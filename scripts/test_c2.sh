timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
export SPCHOL_LIB=$PWD/paper_2409_14009_b200/libspchol.so
python scripts/variant_bench.py --config C2 2>&1 | cut -c1-2000
python scripts/variant_bench.py --config C4 2>&1 | grep lib | cut -c1-300
