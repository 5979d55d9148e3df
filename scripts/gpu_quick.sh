cd /root/repo
export SPCHOL_LIB=$PWD/paper_2409_14009_b200/libspchol.so
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -m gpu -x -q 2>&1 | tail -15 | grep -E "passed|failed|Error|error|assert" | head -20
