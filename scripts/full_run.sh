timeout 1500 python -m pytest tests/ -m gpu -x -q 2>&1 | grep -E "passed|failed|Error|assert" | head -5
for c in C1 C2 C3 C5; do python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['config_id'], round(d['ms_per_step'],2),'ms', round(d['value']/1e3,2),'TF/s', round(d['pct_fp64_peak'],1),'%', 'e2e', round(d['e2e']['seconds_per_step']*1e3,2), 'ms berr', d['e2e']['backward_error'])"; done
python bench.py --steps 5 --warmup 3 2>&1 | tee gpurun_out/bench_full.log | tail -1 | cut -c1-300
