cd /root/repo
export SPCHOL_LIB=$PWD/paper_2409_14009_b200/libspchol.so
mkdir -p gpurun_out
for c in C2 C3 C4; do
  timeout 120 python scripts/solve_bench.py --config $c
  SPCHOL_SOLVE_LEGACY=1 timeout 120 python scripts/solve_bench.py --config $c
done 2>&1 | tee gpurun_out/solve_ab.txt

for c in C4 C5; do timeout 200 python scripts/solve_bench.py --config $c --nrhs 4; done 2>&1 | tee -a gpurun_out/solve_ab.txt
