for f in ${LIBS:-build_variants/*.so}; do
  SPCHOL_LIB=$PWD/$f timeout 120 python -m pytest tests/test_gpu_parity.py -x -q -k "configs" 2>&1 | tail -1
  SPCHOL_LIB=$PWD/$f timeout 120 python scripts/variant_bench.py --config ${CFG:-C4} | grep lib | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['lib'].split('/')[-1], round(d['ms'],2), {k:(v['ms'],v['tf']) for k,v in d['kernels'].items()})"
done
