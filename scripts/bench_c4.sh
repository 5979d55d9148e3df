set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv
python bench.py --config C1 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -3
python bench.py --config C4 --steps 3 --warmup 3 2>&1 | tee gpurun_out/bench_c4.log | tail -5
