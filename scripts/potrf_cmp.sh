for L in paper_2409_14009_b200/libspchol.so build_variants/lib_potrf4.so; do
  export SPCHOL_LIB=$PWD/$L
  python -m pytest tests/test_gpu_parity.py -x -q -k "configs or block" 2>&1 | tail -1
  python scripts/variant_bench.py | grep lib | cut -c1-300
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:potrf -s 480 -c 5 --csv python scripts/profile_factor.py --config C4 2>/dev/null | grep -o '"[0-9.]*"$' | tr '\n' ' '; echo
done
