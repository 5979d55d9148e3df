export SPCHOL_LIB=$PWD/paper_2409_14009_b200/libspchol.so
timeout 900 python -m pytest tests/ -m gpu -x -q 2>&1 | grep -E "passed|failed|^E " | head -5
python - <<'PY'
import json, time, torch, gen, paper_2409_14009_b200 as sp
for c in ["C3", "C4"]:
    p = gen.make(c)
    for um in (0, 1):
        h = sp.Solver.from_problem(p, update_mode=um)
        h.spchol_factor(); h.spchol_factor()
        torch.cuda.synchronize(); t = time.perf_counter()
        for _ in range(3): h.spchol_factor()
        ms = (time.perf_counter() - t) / 3 * 1e3
        h.spchol_enable_kernel_timing(True); h.spchol_factor_async()
        st = h.spchol_kernel_stats("rlb_update" if um else "syrk_scatter")
        print(c, "RLB" if um else "RL", "factor %.2f ms" % ms, "update kernel %.2f ms %.1f TF/s" % (st["ms"], st["flops"] / st["ms"] / 1e9))
        h.close()
PY
