cd /root/repo
export SPCHOL_LIB=$PWD/paper_2409_14009_b200/libspchol.so
mkdir -p gpurun_out
for c in C2 C3 C4; do
  for d in 0 1; do
    timeout 300 python scripts/variant_bench.py --config $c --det $d --vr $([ $d = 1 ] && echo 1 || echo 0) | grep lib | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c det=$d', round(d['ms'],2))"
  done
  timeout 300 python scripts/variant_bench.py --config $c --vr 1 | grep lib | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c det=0 vr=1', round(d['ms'],2))"
done 2>&1 | tee gpurun_out/det_bench.txt
for c in C2 C4; do timeout 600 python bench.py --config $c 2>/dev/null | tail -1 > gpurun_out/bench_$c.json; done
python -c "
import json
for c in ['C2','C4']:
    d=json.load(open('gpurun_out/bench_%s.json'%c)); print(c, d['value'], d['ms_per_step'], d['e2e']['value'], d['e2e'].get('solve_ms'), d['clocks'])"
