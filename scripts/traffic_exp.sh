timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
SPCHOL_LIB=$PWD/paper_2409_14009_b200/libspchol.so python scripts/variant_bench.py | grep lib | cut -c1-400
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --kernel-name-base mangled -k regex:gemm_kernelILi2 --csv --log-file gpurun_out/scatter_dram2.csv python scripts/profile_factor.py --config C4 > /dev/null 2>&1
