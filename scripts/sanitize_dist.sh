#!/bin/bash
# compute-sanitizer memcheck over the multi-rank path (ranks as threads over tests/mock_nccl, per-rank
# VMM arenas) and over the memory-capped mode.  Logs: gpurun_out/sanitizer_dist.log
set -u
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
L=gpurun_out/sanitizer_dist.log
echo "=== memcheck mock 3 ranks S4 (distribution forced, outer 1)" >> $L
SPCHOL_DIST_MINFLOPS=0 SPCHOL_OUTER=1 timeout 1200 $CS --tool memcheck --error-exitcode 9 python tests/mock_dist_run.py S4 3 >> $L 2>&1
echo "exit $?" >> $L
echo "=== memcheck capped S4 (cap 0.6 x arena)" >> $L
timeout 900 $CS --tool memcheck --error-exitcode 9 python -c "
import sys; sys.path.insert(0, '.')
import gen, paper_2409_14009_b200 as sp
p = gen.make('S4')
with sp.Solver.from_problem(p, device=-1) as h0: cap = int(0.6 * h0.query('ARENA_BYTES'))
with sp.Solver.from_problem(p, device_mem_cap=cap, use_graph=0) as h:
    h.spchol_factor(); xs, b = gen.rhs(p); x = h.spchol_solve(b); print('capped berr', gen.backward_error(p, x, b), 'batches', h.query('NBATCHES'))
" >> $L 2>&1
echo "exit $?" >> $L
