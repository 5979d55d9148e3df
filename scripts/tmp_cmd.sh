./tools/panel_probe 2048 > gpurun_out/panel_probe.txt 2>&1
./tools/potrf_probe > gpurun_out/potrf_probe.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fused or parity_configs" > gpurun_out/fused_tests.log 2>&1; echo rc=$? >> gpurun_out/fused_tests.log
timeout 300 python scripts/chain_bench.py 2048 4096 8192 > gpurun_out/chain_now.txt 2>&1
for C in C2 C3 C4; do timeout 600 python bench.py --config $C --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/q_${C}.json 2>/dev/null; echo "$C $(python -c "import json;d=json.loads(open('gpurun_out/q_${C}.json').read().strip().splitlines()[-1]);print(d['ms_per_step'])")" >> gpurun_out/q.txt; done
