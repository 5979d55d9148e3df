"""Model of the multi-GPU schedule (host-only handles, no GPU), per world size W:
  work      critical rank path = max over ranks of phase-A flops + sum over top levels of the max over
            ranks of that level's phase-C flops; bound = whole-factor flops / critical path
  memory    physical device bytes of each rank's arena (own subtree panels, owned top block columns,
            broadcast ring, update and receive regions, inverses) against the single-GPU arena
  traffic   bytes each rank sends / receives per factor: the boundary-block exchange after phase A
            (SURVEY §8(e) phase B), the partial-U exchanges of the top levels, the block-column
            broadcasts; a time estimate at 450 GB/s per direction per GPU (half the NVLink 5 peak)
Writes profiles/r02_dist_model.json."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2409_14009_b200 as sp  # noqa: E402

BW = 450e9


def model(p, W):
    res = []
    for r in range(W):
        with sp.Solver.from_problem(p, device=-1, dist_world=W, dist_rank=r) as h:
            a, lv = h.spchol_dist_plan_flops()
            q = h.query
            res.append(dict(a=a, lv=lv, ntop_dist=q("NTOP_DIST"), markers=q("NMARKERS"), arena=q("ARENA_BYTES"),
                            send=q("COMM_SEND_BYTES"), recv=q("COMM_RECV_BYTES"), b_send=q("COMM_B_SEND_BYTES"),
                            b_recv=q("COMM_B_RECV_BYTES")))
    nl = len(res[0]["lv"])
    crit_a = max(x["a"] for x in res)
    crit_c = sum(max(x["lv"][l] for x in res) for l in range(nl))
    tot = sum(x["a"] + x["lv"].sum() for x in res)
    per = lambda k: [x[k] for x in res]  # noqa: E731
    return dict(bound=tot / (crit_a + crit_c), phase_a_max=crit_a, phase_c_crit=crit_c, ntop_dist=res[0]["ntop_dist"],
                markers=res[0]["markers"], arena_GB=[x / 1e9 for x in per("arena")],
                phaseB_send_GB=[x / 1e9 for x in per("b_send")], phaseB_recv_GB=[x / 1e9 for x in per("b_recv")],
                send_GB=[x / 1e9 for x in per("send")], recv_GB=[x / 1e9 for x in per("recv")],
                comm_ms_at_450GBps=max(max(x["send"], x["recv"]) for x in res) / BW * 1e3)


if __name__ == "__main__":
    cfgs = sys.argv[1:] or ["C3", "C4", "C5"]
    out = {}
    for c in cfgs:
        p = gen.make(c)
        with sp.Solver.from_problem(p, device=-1) as h:
            out[f"{c}/1"] = dict(arena_GB=h.query("ARENA_BYTES") / 1e9, flops_exec=h.query("FLOPS_EXEC"))
        for W in (2, 4, 8):
            m = model(p, W)
            out[f"{c}/{W}"] = m
            print(c, W, json.dumps({k: (round(v, 3) if isinstance(v, float) else
                                        [round(x, 3) for x in v] if isinstance(v, list) else v) for k, v in m.items()}),
                  flush=True)
    os.makedirs("profiles", exist_ok=True)
    json.dump(out, open("profiles/r02_dist_model.json", "w"), indent=1)
