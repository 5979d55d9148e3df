"""Work model of the multi-GPU schedule (host-only handles, no GPU): for each world size, the
critical rank path = max over ranks of phase-A flops + sum over top levels of the max over ranks of
that level's phase-C flops; bound = whole-factor flops / critical path.  Compares the distributed top
(default) with the fan-in schedule (SPCHOL_DIST_MINFLOPS=inf: every top supernode on one rank)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2409_14009_b200 as sp  # noqa: E402


def model(p, W):
    res = []
    for r in range(W):
        with sp.Solver.from_problem(p, device=-1, dist_world=W, dist_rank=r) as h:
            res.append(h.spchol_dist_plan_flops() + (h.query("NTOP_DIST"), h.query("NMARKERS")))
    nl = len(res[0][1])
    crit_a = max(a for a, *_ in res)
    crit_c = sum(max(x[1][l] for x in res) for l in range(nl))
    tot = sum(a + lv.sum() for a, lv, *_ in res)
    return dict(bound=tot / (crit_a + crit_c), phase_a_max=crit_a, phase_c_crit=crit_c, ntop_dist=res[0][2],
                markers=res[0][3])


if __name__ == "__main__":
    cfgs = sys.argv[1:] or ["C3", "C4", "C5"]
    out = {}
    for c in cfgs:
        p = gen.make(c)
        for mode, env in (("distributed", None), ("fan-in", "1e300")):
            if env:
                os.environ["SPCHOL_DIST_MINFLOPS"] = env
            else:
                os.environ.pop("SPCHOL_DIST_MINFLOPS", None)
            for W in (2, 4, 8):
                m = model(p, W)
                out[f"{c}/{mode}/{W}"] = m
                print(c, mode, W, json.dumps({k: (round(v, 3) if isinstance(v, float) and v < 1e3 else v) for k, v in m.items()}), flush=True)
    json.dump(out, open("profiles/r01_dist_work_model.json", "w"), indent=1)
