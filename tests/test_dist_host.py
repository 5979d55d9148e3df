"""Multi-GPU host-side logic on CPU: gloo processes build host-only handles for their ranks and check
that the subtree-to-GPU mapping is identical on every rank, partitions the supernodes
into whole subtrees plus a top that is closed under ancestors, lays each rank's subtree panels out
as one region below the top panels, and that every rank's plan holds the same marker sequence and
matching exchange volumes (what one rank sends, the others receive)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import gen
import paper_2409_14009_b200 as sp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        p = gen.make(name)
        with sp.Solver.from_problem(p, device=-1, dist_world=world, dist_rank=rank) as h:
            owner, top_off, top_slot = h.spchol_export_mapping()
            sym = h.spchol_export_symbolic()
            off, ld, _ = h.spchol_export_panels(values=False)
            h_send, h_recv = h.query("COMM_SEND_BYTES"), h.query("COMM_RECV_BYTES")
        t = torch.from_numpy(owner.astype(np.int64))
        got = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(got, t)
        for g in got:
            assert torch.equal(g, t), "ranks disagree on the mapping"
        sparent = sym["sparent"]
        ns = len(sparent)
        # whole subtrees: a local supernode's parent is local to the same rank or top
        for J in range(ns):
            P = sparent[J]
            if P >= 0 and owner[P] >= 0:
                assert owner[J] == owner[P]
            if owner[J] < 0 and P >= 0:
                assert owner[P] < 0, "top is closed under ancestors"
        assert set(np.unique(owner[owner >= 0]).tolist()) <= set(range(world))
        # per-rank arena layout: rank q's subtree panels form one region, all below the top panels
        k = np.diff(sym["sfirst"])
        sizes = ld.astype(np.int64) * k
        top = owner < 0
        if top.any():
            assert off[:-1][top].min() >= top_off
        for rq in range(world):
            mine = owner == rq
            if mine.any() and (owner > rq).any():
                assert (off[:-1][mine] + sizes[mine]).max() <= off[:-1][owner > rq].min()
        if (~top).any():
            assert (off[:-1][~top] + sizes[~top]).max() <= top_off
        # exchange volumes: the bytes all ranks send equal the bytes all ranks receive
        vol = torch.tensor([h_send, h_recv], dtype=torch.float64)
        dist.all_reduce(vol)
        assert vol[0].item() == vol[1].item()
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok", int(top.sum()), [int((owner == r).sum()) for r in range(world)]))
    except Exception as e:  # noqa: BLE001
        q.put((rank, f"error: {e!r}", 0, []))


@pytest.mark.parametrize("name,world", [("S4", 2), ("C1", 2), ("S5", 2), ("S2", 3), ("S4", 4)])
def test_mapping_two_process_gloo(name, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
    for r in res:
        assert r[1] == "ok", r
    # every rank owns at least one subtree
    assert all(c > 0 for c in res[0][3])


def test_mapping_single_process_properties():
    p = gen.make("C1")
    for W in (2, 4, 8):
        with sp.Solver.from_problem(p, device=-1, dist_world=W, dist_rank=W - 1) as h:
            owner, towner, top_off, top_slot = h.spchol_export_mapping(with_top_owner=True)
            assert (owner < 0).any() and all((owner == r).any() for r in range(W))
            # every top supernode has an owner rank; subtree supernodes have none
            assert np.all((towner >= 0) == (owner < 0)) and towner.max() < W
    with sp.Solver.from_problem(p, device=-1) as h:
        owner, top_off, _ = h.spchol_export_mapping()
        assert (owner == 0).all() and top_off == h.query("PANEL_DOUBLES")
    with pytest.raises(sp.SpcholError):
        sp.Solver.from_problem(p, device=-1, dist_world=2, dist_rank=2)


def _plan_work(p, W, r, **opts):
    with sp.Solver.from_problem(p, device=-1, dist_world=W, dist_rank=r, **opts) as h:
        a, lv = h.spchol_dist_plan_flops()
        return (a, lv, h.query("NMARKERS"), h.query("NTOP_DIST"), h.query("FLOPS_EXEC"), h.query("COMM_SEND_BYTES"),
                h.query("COMM_RECV_BYTES"), h.query("ARENA_BYTES"))


@pytest.mark.parametrize("name,minflops,outer", [("S4", "0", None), ("S5", "0", "1"), ("C1", "0", "1"),
                                                  ("S4", None, None), ("S2", "0", "1")])
def test_distributed_top_plan_partitions_work(name, minflops, outer, monkeypatch):
    """Distributed top (block-column cyclic cdiv, K-split partial U_J): every flop of the single-GPU
    plan runs on exactly one rank — the executed flops of all ranks' plans (phase A + phase C) add up
    to the whole factor's — all ranks hold the same number of exchange markers, the bytes sent equal
    the bytes received (the per-rank arena is checked at full size: 2 MB pages dominate here)."""
    if minflops is not None:
        monkeypatch.setenv("SPCHOL_DIST_MINFLOPS", minflops)
    if outer is not None:
        monkeypatch.setenv("SPCHOL_OUTER", outer)
    p = gen.make(name)
    # every supernode on the blocked path on both sides (multi-GPU top supernodes always are), so the
    # per-launch flop accounting is the same
    with sp.Solver.from_problem(p, device=-1, small_max_k=-1) as h:
        whole, _ = h.spchol_dist_plan_flops()
    for W in (2, 3, 4, 8):
        res = [_plan_work(p, W, r, small_max_k=-1) for r in range(W)]
        tot = sum(a + lv.sum() for a, lv, *_ in res)
        assert abs(tot - whole) <= 1e-9 * whole, (W, tot, whole)
        assert len({r_[2] for r_ in res}) == 1
        assert sum(r_[5] for r_ in res) == sum(r_[6] for r_ in res)
        if minflops == "0" and name != "C1":     # C1's top supernodes are below one outer block
            assert res[0][3] > 0
        # distributing the top never makes the critical rank path longer than the fan-in schedule
        crit = max(a for a, *_ in res) + sum(max(r_[1][l] for r_ in res) for l in range(len(res[0][1])))
        assert crit <= whole


@pytest.mark.slow
@pytest.mark.parametrize("name", ["C4", "C5"])
def test_fullsize_distribution_model(name):
    """The north_star configs' multi-GPU plans (host-only, the driver's 2/4/8-GPU runs): exact work
    partition, per-rank arena well below the single-GPU one, and the work model's speedup bound
    (max over ranks of phase A + per top level max over ranks) above 6x at 8 ranks on C4."""
    p = gen.make(name)
    with sp.Solver.from_problem(p, device=-1) as h:
        whole, _ = h.spchol_dist_plan_flops()
        arena1 = h.query("ARENA_BYTES")
    for W in (2, 4, 8):
        res = [_plan_work(p, W, r) for r in range(W)]
        assert abs(sum(a + lv.sum() for a, lv, *_ in res) - whole) <= 1e-9 * whole
        crit = max(a for a, *_ in res) + sum(max(r_[1][l] for r_ in res) for l in range(len(res[0][1])))
        if name == "C4" and W == 8:
            assert whole / crit >= 6.0, whole / crit
        assert max(r_[7] for r_ in res) <= arena1 * (1.5 / W + 0.2)


def test_bench_dry_run_two_ranks():
    """`bench.py --dry-run --gpus N` (no GPU): every rank's host-only plan, the same marker count on all
    ranks and an exact partition of the single-GPU work."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for n in (2, 4):
        out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--dry-run", "--gpus", str(n),
                              "--config", "S4"], capture_output=True, text=True, timeout=300, check=True).stdout
        d = json.loads([ln for ln in out.splitlines() if ln.startswith("{")][-1])
        assert d["n_gpus"] == n and len(d["ranks"]) == n
        assert d["markers_match"] and d["work_partition_exact"]
