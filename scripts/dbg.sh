timeout 1200 python -m pytest tests/ -m gpu -x -q -s 2>&1 | tail -15
python bench.py --config C2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -5 | cut -c1-800
