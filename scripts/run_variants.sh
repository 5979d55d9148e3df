for f in ${LIBS:-build_variants/*.so}; do SPCHOL_LIB=$PWD/$f python scripts/variant_bench.py --config ${CFG:-C4}; done 2>&1 | grep lib | cut -c1-420
