export SPCHOL_LIB=$PWD/paper_2409_14009_b200/libspchol.so
python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
python scripts/variant_bench.py
