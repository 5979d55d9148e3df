#!/usr/bin/env python
"""Benchmark: numeric RL supernodal Cholesky factorization (arXiv 2409.14009) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl ours|reference]

A "step" is one numeric factorization (panel init, per-level POTRF,
TRSM, SYRK/GEMM + relind scatter) of the config's matrix, with A's values already resident in HBM.
Metric (BASELINE.json): numeric factor time and FP64 GFLOP/s = F_exact / factor time, where
F_exact = sum_j cc_j^2 over the exact factor (padding flops excluded), and % of FP64 peak.

N > 1 (torchrun, one process per GPU): the distributed factorization of ONE matrix (strong
scaling): proportional subtree-to-GPU mapping, each rank factors its subtrees, the top panels are
summed with an NCCL all-reduce, the top supernodes are factored; value = F_exact /
max-over-ranks time.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import gen  # noqa: E402

FP64_PEAK_FILE = os.path.join(ROOT, "profiles", "fp64_peak.json")
TRAFFIC_FILE = os.path.join(ROOT, "profiles", "roofline_traffic.json")
# bounded CPU samples: leading principal block of the ND-ordered matrix (whole ND subtrees)
# Bounded CPU samples (leading principal blocks of the ND-ordered matrix = whole ND subtrees): about
# 1e11 flop for cpu_baseline (C4: 125000 columns = one octant subtree, 1.0e11 flop); the reference
# arm's per-step sample is smaller when many steps are requested (the whole run stays in minutes).
CPU_SAMPLE_COLS = {"C1": 900, "C2": 1000000, "C3": 100000, "C4": 125000, "C5": 60000}
REF_STEP_COLS = {"C1": 900, "C2": 1000000, "C3": 100000, "C4": 125000, "C5": 60000}
REF_STEP_COLS_MANY = {"C1": 900, "C2": 400000, "C3": 40000, "C4": 60000, "C5": 30000}


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def fp64_peak():
    """Measured FP64 DMMA peak (tools/fp64_peak.cu on this pool's B200, profiles/fp64_peak.json)."""
    with open(FP64_PEAK_FILE) as f:
        d = json.load(f)
    return d


class Clocks:
    """Clock / throttle-reason sampling during the timed region (B200_PROFILING.md recipe): NVML
    (pynvml) polled every 2 ms from a thread, so even a ~50 ms timed region gets samples;
    nvidia-smi -lms 100 when NVML is unavailable."""

    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index):
        self.index = index
        self.p = None
        self.samples = []
        self.nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.bits = [pynvml.nvmlClocksEventReasonHwSlowdown, pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                         pynvml.nvmlClocksEventReasonSwThermalSlowdown, pynvml.nvmlClocksEventReasonSwPowerCap]
        except Exception:  # noqa: BLE001
            self.nvml = None

    def _poll(self):
        nv = self.nvml
        while not self.stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                mx = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append([str(sm), str(mx), ""] + ["Active" if r & b else "Not Active" for b in self.bits])
            except Exception:  # noqa: BLE001
                pass
            self.stop.wait(0.002)

    def __enter__(self):
        self.samples = []
        if self.nvml is not None:
            import threading
            self.stop = threading.Event()
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return self
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self.p = None
        return self

    def __exit__(self, *a):
        if self.nvml is not None:
            self.stop.set()
            self.t.join(timeout=5)
            return
        if self.p is None:
            return
        time.sleep(0.25)
        self.p.terminate()
        out, _ = self.p.communicate(timeout=10)
        for line in out.strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                self.samples.append(parts)

    def summary(self):
        if not getattr(self, "samples", None):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        reasons = sorted({self.NAMES[i] for s in self.samples for i in range(4) if s[3 + i].lower() == "active"})
        loaded = [x for x in sm if x > 0.5 * max(sm)] if sm else []
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples),
                "source": "nvml" if self.nvml is not None else "nvidia-smi"}


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def self_launch(args):
    """`bench.py --gpus N` (N > 1) started without a launcher: re-run this script under
    torch.distributed.run with N local ranks (one process per GPU) and return its exit code."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def run_reference(args):
    """--impl reference: the CPU oracle (as it stands) on the host cores, a bounded sample per step."""
    import oracle
    world, rank, _ = dist_setup(args)
    if rank != 0:
        return
    prob = gen.make(args.config)
    cols = REF_STEP_COLS if args.steps + args.warmup <= 8 else REF_STEP_COLS_MANY
    ns = min(prob.n, cols.get(args.config, 20000))
    sub = gen.leading_submatrix(prob, ns)
    o = oracle.Oracle.from_problem(sub)
    cores = host_cores()
    for _ in range(args.warmup):
        o.factor(threads=cores)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        fc = o.factor(threads=cores)
        times.append(time.perf_counter() - t0)
        assert fc == -1
    t = sum(times) / len(times)
    gflops = o.flops / t / 1e9
    sample = (f"leading {ns}x{ns} principal block (whole ND subtrees) of {args.config}'s ND-ordered matrix "
              f"(F_exact {o.flops:.4g} flop), level-parallel oracle build (bit-identical to serial) on {cores} threads")
    line = {
        "impl": "reference", "metric": "numeric factor FP64 GFLOP/s (F_exact / factor time)", "value": gflops,
        "unit": "GFLOP/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": gen.CONFIGS[args.config]["desc"], "sample": sample},
        "cpu_baseline": {"value": gflops, "unit": "GFLOP/s", "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": gflops, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(args, seconds_hint=True):
    import oracle
    prob = gen.make(args.config)
    ns = min(prob.n, CPU_SAMPLE_COLS.get(args.config, 30000))
    sub = gen.leading_submatrix(prob, ns)
    o = oracle.Oracle.from_problem(sub)
    cores = host_cores()
    t0 = time.perf_counter()
    fc = o.factor(threads=cores)
    t = time.perf_counter() - t0
    assert fc == -1
    return {"value": o.flops / t / 1e9, "unit": "GFLOP/s", "cores": cores, "kind": "oracle",
            "sample": f"leading {ns}x{ns} principal block (whole ND subtrees) of {args.config}'s ND-ordered matrix "
                      f"(F_exact {o.flops:.4g} flop, {t:.1f} s), level-parallel oracle build (bit-identical to the "
                      f"serial one) on {cores} threads"}


def dry_run(args):
    """Host-only plans of all N ranks (the multi-GPU schedule without a GPU): per rank the executed
    flops of phase A and phase C, exchange markers, per-rank arena and communication volume; checks
    that the ranks' plans pair up (same marker count) and partition the single-GPU work."""
    import paper_2409_14009_b200 as sp
    prob = gen.make(args.config)
    with sp.Solver.from_problem(prob, device=-1) as h:
        whole, _ = h.spchol_dist_plan_flops()
        arena1 = h.query("ARENA_BYTES")
    ranks = []
    for r in range(args.gpus):
        with sp.Solver.from_problem(prob, device=-1, dist_world=args.gpus, dist_rank=r) as h:
            a, lv = h.spchol_dist_plan_flops()
            ranks.append({"rank": r, "phase_a_flops": a, "phase_c_flops": float(lv.sum()), "level_flops": lv.tolist(),
                          "markers": h.query("NMARKERS"), "arena_GB": h.query("ARENA_BYTES") / 1e9,
                          "send_GB": h.query("COMM_SEND_BYTES") / 1e9, "recv_GB": h.query("COMM_RECV_BYTES") / 1e9,
                          "top_distributed": h.query("NTOP_DIST")})
    nl = len(ranks[0]["level_flops"])
    crit = max(x["phase_a_flops"] for x in ranks) + sum(max(x["level_flops"][l] for x in ranks) for l in range(nl))
    tot = sum(x["phase_a_flops"] + x["phase_c_flops"] for x in ranks)
    for x in ranks:
        del x["level_flops"]
    print(json.dumps({"dry_run": True, "config": args.config, "n_gpus": args.gpus,
                      "markers_match": len({x["markers"] for x in ranks}) == 1,
                      "work_partition_exact": abs(tot - whole) <= 1e-9 * whole,
                      "work_model_speedup": whole / crit, "single_gpu_arena_GB": arena1 / 1e9, "ranks": ranks}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C4", choices=sorted(gen.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--dry-run", action="store_true",
                    help="no GPU: build every rank's host-only plan for --gpus N and print the schedule model")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference(args)
        return
    if args.dry_run:
        dry_run(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    if int(os.environ.get("WORLD_SIZE", "1")) != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={os.environ.get('WORLD_SIZE')}")

    import torch
    import paper_2409_14009_b200 as sp

    world, rank, local = dist_setup(args)
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.cuda.current_device()
    prob = gen.make(args.config)
    t0 = time.perf_counter()
    dist_mode = "1 GPU"
    if world > 1:
        # distributed factor of ONE matrix over the ranks; any setup failure ends the run (non-zero
        # exit) — there is no replica fallback
        h = sp.Solver.from_problem(prob, device=dev, dist_world=world, dist_rank=rank)
        uid = [sp.spchol_dist_nccl_unique_id() if rank == 0 else None]
        torch.distributed.broadcast_object_list(uid, src=0)
        h.spchol_dist_attach_nccl(uid[0])
        dist_mode = (f"subtree-to-GPU x{world}: proportional mapping of the supernodal etree, top supernodes "
                     f"distributed over their rank groups, NCCL exchanges")
    else:
        h = sp.Solver.from_problem(prob, device=dev)
    analyze_s = time.perf_counter() - t0
    stream = torch.cuda.Stream()
    h.spchol_set_stream(stream.cuda_stream)
    F = float(h.query("FLOPS_EXACT"))
    Fexec = float(h.query("FLOPS_EXEC"))
    launches_per_step = h.query("LAUNCHES")

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    # ---- warm-up (graph capture happens on the first factor)
    for _ in range(args.warmup):
        h.spchol_factor()
    # ---- timed region: K factorizations, device-resident values; inputs (13.5 GB panels on C4)
    # are far larger than the 126 MB L2, so no explicit flush is needed between steps.
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    with Clocks(dev) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            h.spchol_factor_async()
        ev1.record(stream)
        barrier()
    fc, _ = h.spchol_factor_status()
    assert fc == -1
    ms = max_over_ranks(ev0.elapsed_time(ev1) / args.steps)
    value = F / (ms / 1e3) / 1e9   # distributed: one matrix (strong scaling)
    peak = fp64_peak()

    # ---- roofline of the dominant kernel (SYRK/GEMM + relind scatter), CUDA events per launch
    h.spchol_enable_kernel_timing(True)
    barrier()
    for _ in range(args.steps):
        h.spchol_factor_async()
    barrier()
    stats = {k: h.spchol_kernel_stats(k) for k in sp.KERNEL_KINDS}
    h.spchol_enable_kernel_timing(False)
    # dominant kernel = the class carrying the most flops (event timings of tiny launches in this
    # serialized pass include host submission gaps, so "most milliseconds" misleads on C2/C3)
    dom = max(stats, key=lambda k: stats[k]["flops"])
    sd = stats[dom]
    achieved = sd["flops"] / (sd["ms"] / 1e3) / 1e12 if sd["ms"] > 0 else 0.0
    traffic = None
    if os.path.exists(TRAFFIC_FILE):
        # ncu-measured DRAM bytes per launch of the dominant kernel (profiles/roofline_traffic.json),
        # used only while the kernel source is the one it was measured on (else null, not stale)
        import hashlib
        with open(TRAFFIC_FILE) as f:
            tr = json.load(f)
        with open(os.path.join(ROOT, "paper_2409_14009_b200", "csrc", "kernels.cu"), "rb") as f:
            same_src = hashlib.sha256(f.read()).hexdigest() == tr.get("kernels_cu_sha256")
        if tr.get("config") == args.config and tr.get("kernel") == dom and same_src:
            traffic = tr.get("traffic_bytes_per_launch")
    step_ms_timed = sum(v["ms"] for v in stats.values()) / args.steps
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peak["dmma_tflops_burst"], "unit": "TFLOP/s",
                "frac": achieved / peak["dmma_tflops_burst"], "traffic": traffic, "kernel": dom,
                "kernel_share_of_step": sd["ms"] / args.steps / step_ms_timed if step_ms_timed else None,
                "launches_per_step": sd["launches"] // args.steps,
                "peak_source": "measured FP64 DMMA m8n8k4 microbenchmark on this pool's B200 "
                               "(profiles/fp64_peak.json; MEASURED_PEAKS.json has no FP64 entry)",
                "per_kernel_ms_per_step": {k: v["ms"] / args.steps for k, v in stats.items()},
                "per_kernel_tflops": {k: (v["flops"] / (v["ms"] / 1e3) / 1e12 if v["ms"] > 0 and v["flops"] > 0 else None)
                                      for k, v in stats.items()},
                # algorithmic bytes / time of each class (the HBM roofline of a1 init, the small
                # kernels and the assembly; 6539 GB/s measured copy bandwidth, MEASURED_PEAKS.json)
                "per_kernel_GBps": {k: (v["bytes"] / (v["ms"] / 1e3) / 1e9 if v["ms"] > 0 and v["bytes"] > 0 else None)
                                    for k, v in stats.items()}}

    # ---- end to end through the public API with host buffers (pinned): H2D of A's values and b,
    # factor, solve, D2H of x — every step.
    e2e = None
    if not args.no_e2e:
        vals_h = torch.from_numpy(prob.values).pin_memory()
        xs, b = gen.rhs(prob)
        b_h = torch.from_numpy(b).pin_memory()
        x_h = torch.empty_like(b_h).pin_memory()
        L = sp.lib()
        import ctypes
        vp = ctypes.c_void_p
        def e2e_step():
            assert L.spchol_set_values(h._h, vp(vals_h.data_ptr())) == 0
            assert L.spchol_factor(h._h, None, None) == 0
            assert L.spchol_solve(h._h, vp(b_h.data_ptr()), vp(x_h.data_ptr()), 1, prob.n) == 0
        e2e_step()
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_step()
        barrier()
        e2e_s = max_over_ranks((time.perf_counter() - t0) / args.steps)
        berr = gen.backward_error(prob, x_h.numpy(), b)   # verification only, not timed
        # solve alone (device-resident b and x, CUDA events): SURVEY §8(f-1)
        d_b = torch.from_numpy(b).to(dev)
        d_x = torch.empty_like(d_b)
        for _ in range(2):
            h.spchol_solve_device(d_b.data_ptr(), d_x.data_ptr())
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        s0.record(stream)
        for _ in range(args.steps):
            h.spchol_solve_device(d_b.data_ptr(), d_x.data_ptr())
        s1.record(stream)
        barrier()
        solve_ms = max_over_ranks(s0.elapsed_time(s1) / args.steps)
        e2e = {"solve_ms": solve_ms, "solve_GBps_L_read_twice": 2 * 8 * h.query("NNZ_L") / (solve_ms / 1e3) / 1e9,
               "value": F / e2e_s / 1e9, "unit": "GFLOP/s", "h2d_bytes_per_step": 8 * (prob.nnz + prob.n),
               "d2h_bytes_per_step": 8 * prob.n + 8, "seconds_per_step": e2e_s, "includes": "set_values(H2D) + factor + solve(H2D b, D2H x)",
               "backward_error": berr}

    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return
    cpu = None if args.no_cpu_baseline or world > 1 else cpu_baseline(args)
    line = {
        "metric": "numeric factor FP64 GFLOP/s (F_exact / factor time)",
        "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": gen.CONFIGS[args.config]["desc"], "config_id": args.config, "n": prob.n,
                   "nnz_A_lower": prob.nnz, "nnz_L": h.query("NNZ_L"), "flops_exact": F, "flops_executed": Fexec,
                   "supernodes": h.query("NSUPER"), "levels": h.query("NLEVELS"),
                   "panel_GB": h.query("PANEL_DOUBLES") * 8 / 1e9, "analyze_s": analyze_s,
                   "l2": "no flush needed: panels (GB) >> 126 MB L2",
                   "parallelism": dist_mode},
        "factor_s": ms / 1e3,
        "pct_fp64_peak": 100.0 * (F / (ms / 1e3) / 1e12) / peak["dmma_tflops_burst"],
        "clocks": clk.summary(),
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches_per_step * args.steps,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
