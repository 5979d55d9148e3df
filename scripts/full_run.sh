set -x
timeout 1500 python -m pytest tests/ -m gpu -x -q -s 2>&1 | grep -E "passed|failed|Error|logdet|assert" | head -30
for c in C2 C3 C5; do python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-600; done
python bench.py --steps 5 --warmup 3 2>&1 | tee gpurun_out/bench_full.log | tail -1
