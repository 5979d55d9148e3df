set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests/ -m gpu -q -x 2>&1 | tail -15
timeout 600 python bench.py --steps 5 --warmup 3 2>gpurun_out/bench_C4.err | tail -1 > gpurun_out/bench_C4.json
for c in C2 C3; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/bench_$c.json; done
cat gpurun_out/bench_C*.json | cut -c1-400
