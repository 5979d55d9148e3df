# usage: bash scripts/ms.sh CONFIG [env assignments...] -> prints the factor ms of variant_bench
c=$1; shift
env "$@" python scripts/variant_bench.py --config $c | grep '"lib"' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', '$*', round(d['ms'],2))"
