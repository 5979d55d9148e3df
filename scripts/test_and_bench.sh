set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -5
python bench.py --config ${CFG:-C4} --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tee gpurun_out/bench.log | tail -3
