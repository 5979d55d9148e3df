"""B200-native right-looking supernodal sparse Cholesky (RL, arXiv 2409.14009).

Thin ctypes binding over ``libspchol.so`` (the C ABI in ``include/spchol.h``): argument
marshalling only — every step of analyze / factor / solve runs in the library (host symbolic
analysis in C++, the numeric factorization and solves in sm_100a CUDA kernels).  There is no
CPU fallback: if the library is missing this module raises on import of :func:`lib`.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SPCHOL_LIB") or os.path.join(_HERE, "libspchol.so")
_LIB = None

SPCHOL_OK = 0
SPCHOL_ERR_DIMENSION = -1
SPCHOL_ERR_VALIDATION = -2
SPCHOL_ERR_NOT_SPD = -3
SPCHOL_ERR_DEVICE_OOM = -4
SPCHOL_ERR_CUDA = -5
SPCHOL_ERR_NCCL = -6
SPCHOL_ERR_STATE = -7

Q = dict(N=0, NNZ_A=1, NNZ_L=2, NFUND=3, NSUPER=4, ADDED=5, NLEVELS=6, ROWS_LEN=7, NPAIRS=8,
         RELIND_LEN=9, PANEL_DOUBLES=10, NMERGES=11, FLOPS_EXACT=12, FLOPS_EXEC=13, LAUNCHES=14,
         UPDATE_ENTRIES=15, NBLOCKS=16, NMARKERS=17, NTOP_DIST=18, DEVICE_BYTES=19, COMM_SEND_BYTES=20,
         COMM_RECV_BYTES=21, ARENA_BYTES=22, DIST_GRAPH=23, COMM_B_SEND_BYTES=24, COMM_B_RECV_BYTES=25, NBATCHES=26,
         HOST_BYTES=27)
KERNEL_KINDS = dict(small=0, potrf=1, trsm=2, local_update=3, syrk_scatter=4, init=5, rlb_update=6, panel=7)

# Every symbol include/spchol.h declares (checked by tests/test_capi_exports.py).
EXPORTS = [
    "spchol_default_options", "spchol_analyze", "spchol_save_analysis", "spchol_load_analysis",
    "spchol_export_factor_csc", "spchol_set_values", "spchol_set_values_device",
    "spchol_set_stream", "spchol_factor_async", "spchol_factor_status", "spchol_factor",
    "spchol_solve", "spchol_solve_device", "spchol_query", "spchol_export_symbolic",
    "spchol_export_blocks", "spchol_export_panels", "spchol_export_panel", "spchol_export_diagonal", "spchol_enable_kernel_timing", "spchol_kernel_stats",
    "spchol_kernel_trace", "spchol_dist_init", "spchol_dist_nccl_unique_id", "spchol_dist_attach_nccl",
    "spchol_export_mapping",
    "spchol_dist_plan_flops",
    "spchol_destroy", "spchol_last_error",
]


class spchol_options(ctypes.Structure):
    _fields_ = [("merge_cap", ctypes.c_double), ("device", ctypes.c_int32), ("block", ctypes.c_int32),
                ("small_max_k", ctypes.c_int32), ("use_graph", ctypes.c_int32),
                ("dist_rank", ctypes.c_int32), ("dist_world", ctypes.c_int32),
                ("subtree_streams", ctypes.c_int32), ("update_mode", ctypes.c_int32),
                ("deterministic", ctypes.c_int32), ("partition_refinement", ctypes.c_int32), ("device_mem_cap", ctypes.c_int64)]


class SpcholError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"spchol error {code}: {msg}")
        self.code = code


class NotSPDError(SpcholError):
    def __init__(self, code, msg, fail_col, fail_col_orig):
        super().__init__(code, msg)
        self.fail_col = fail_col
        self.fail_col_orig = fail_col_orig


def lib():
    """Load libspchol.so (fails loudly when the CUDA library has not been built)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        vp, i64, i32, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double
        L.spchol_default_options.argtypes = [ctypes.POINTER(spchol_options)]
        L.spchol_default_options.restype = None
        L.spchol_analyze.argtypes = [i64, vp, vp, vp, vp, ctypes.POINTER(spchol_options), ctypes.POINTER(vp)]
        L.spchol_set_values.argtypes = [vp, vp]
        L.spchol_save_analysis.argtypes = [vp, ctypes.c_char_p]
        L.spchol_export_factor_csc.argtypes = [vp, vp, vp, vp, vp]
        L.spchol_load_analysis.argtypes = [ctypes.c_char_p, ctypes.POINTER(spchol_options), ctypes.POINTER(vp)]
        L.spchol_set_values_device.argtypes = [vp, vp]
        L.spchol_set_stream.argtypes = [vp, vp]
        L.spchol_factor_async.argtypes = [vp]
        L.spchol_factor_status.argtypes = [vp, ctypes.POINTER(i64), ctypes.POINTER(i64)]
        L.spchol_factor.argtypes = [vp, ctypes.POINTER(i64), ctypes.POINTER(i64)]
        L.spchol_solve.argtypes = [vp, vp, vp, i32, i64]
        L.spchol_solve_device.argtypes = [vp, vp, vp, i32, i64, vp]
        L.spchol_dist_init.argtypes = [i32, i32, vp]
        L.spchol_query.argtypes = [vp, ctypes.c_int, ctypes.POINTER(i64)]
        L.spchol_export_symbolic.argtypes = [vp] * 19
        L.spchol_export_panels.argtypes = [vp, vp, vp, vp]
        L.spchol_export_blocks.argtypes = [vp] * 6
        L.spchol_export_panel.argtypes = [vp, i32, vp]
        L.spchol_export_diagonal.argtypes = [vp, vp]
        L.spchol_enable_kernel_timing.argtypes = [vp, ctypes.c_int]
        L.spchol_kernel_stats.argtypes = [vp, ctypes.c_int, ctypes.POINTER(i64), ctypes.POINTER(dbl),
                                          ctypes.POINTER(dbl), ctypes.POINTER(dbl)]
        L.spchol_kernel_trace.argtypes = [vp, i64, ctypes.POINTER(i64), vp, vp, vp, vp]
        L.spchol_dist_nccl_unique_id.argtypes = [vp]
        L.spchol_dist_attach_nccl.argtypes = [vp, vp]
        L.spchol_export_mapping.argtypes = [vp, vp, vp, ctypes.POINTER(i64), ctypes.POINTER(i64)]
        L.spchol_dist_plan_flops.argtypes = [vp, ctypes.POINTER(dbl), vp]
        L.spchol_destroy.argtypes = [vp]
        L.spchol_destroy.restype = None
        L.spchol_last_error.argtypes = []
        L.spchol_last_error.restype = ctypes.c_char_p
        for nm in EXPORTS:
            if nm not in ("spchol_default_options", "spchol_destroy", "spchol_last_error"):
                getattr(L, nm).restype = ctypes.c_int
        _LIB = L
    return _LIB


def _vp(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def _check(rc):
    if rc != SPCHOL_OK:
        raise SpcholError(rc, lib().spchol_last_error().decode())
    return rc


def default_options(**kw):
    o = spchol_options()
    lib().spchol_default_options(ctypes.byref(o))
    for k, v in kw.items():
        setattr(o, k, v)
    return o


class Solver:
    """One spchol handle: ``analyze`` on construction, then ``factor`` / ``solve``.

    ``device=-1`` builds a host-only handle (symbolic analysis + launch plan, no GPU).
    """

    def __init__(self, n, colptr, rowidx, values=None, perm=None, _load=None, **options):
        L = lib()
        self._L = L
        if _load is not None:             # spchol_load_analysis
            self.options = default_options(**options)
            h = ctypes.c_void_p()
            _check(L.spchol_load_analysis(str(_load).encode(), ctypes.byref(self.options), ctypes.byref(h)))
            self._h = h
            self.n = self.spchol_query("N")
            self.nnzA = self.spchol_query("NNZ_A")
            return
        colptr = np.ascontiguousarray(colptr, np.int64)
        rowidx = np.ascontiguousarray(rowidx, np.int32)
        vals = None if values is None else np.ascontiguousarray(values, np.float64)
        pm = None if perm is None else np.ascontiguousarray(perm, np.int32)
        self.n = int(n)
        self.nnzA = int(colptr[-1]) if len(colptr) else 0
        self.options = default_options(**options)
        h = ctypes.c_void_p()
        rc = L.spchol_analyze(self.n, _vp(colptr), _vp(rowidx), _vp(vals), _vp(pm), ctypes.byref(self.options),
                              ctypes.byref(h))
        _check(rc)
        self._h = h

    @classmethod
    def spchol_load_analysis(cls, path, **options):
        return cls(0, None, None, _load=path, **options)

    def spchol_export_factor_csc(self, values=True):
        """(Lp int64[n+1], Li int32[nnz(L)], Lx float64[nnz(L)] or None, padding_nonzeros or None)."""
        Lp = np.empty(self.n + 1, np.int64)
        _check(self._L.spchol_export_factor_csc(self._h, _vp(Lp), None, None, None))
        Li = np.empty(int(Lp[-1]), np.int32)
        Lx = np.empty(int(Lp[-1]), np.float64) if values else None
        npad = ctypes.c_int64(-1)
        _check(self._L.spchol_export_factor_csc(self._h, _vp(Lp), _vp(Li), _vp(Lx) if values else None,
                                                ctypes.byref(npad) if values else None))
        return Lp, Li, Lx, (int(npad.value) if values else None)

    def spchol_save_analysis(self, path):
        _check(self._L.spchol_save_analysis(self._h, str(path).encode()))

    @classmethod
    def from_problem(cls, prob, with_values=True, **options):
        return cls(prob.n, prob.colptr, prob.rowidx, prob.values if with_values else None, prob.perm, **options)

    def close(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._L.spchol_destroy(h)
        self._h = None

    __del__ = close

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # ---- C ABI mirrors (same names)
    def spchol_set_values(self, values):
        v = np.ascontiguousarray(values, np.float64)
        assert v.size == self.nnzA
        _check(self._L.spchol_set_values(self._h, _vp(v)))

    def spchol_set_values_device(self, dev_ptr: int):
        _check(self._L.spchol_set_values_device(self._h, ctypes.c_void_p(dev_ptr)))

    def spchol_set_stream(self, stream_ptr: int | None):
        _check(self._L.spchol_set_stream(self._h, ctypes.c_void_p(stream_ptr) if stream_ptr else None))

    def spchol_factor_async(self):
        _check(self._L.spchol_factor_async(self._h))

    def spchol_factor_status(self):
        fc, fo = ctypes.c_int64(-1), ctypes.c_int64(-1)
        rc = self._L.spchol_factor_status(self._h, ctypes.byref(fc), ctypes.byref(fo))
        if rc == SPCHOL_ERR_NOT_SPD:
            raise NotSPDError(rc, self._L.spchol_last_error().decode(), int(fc.value), int(fo.value))
        _check(rc)
        return int(fc.value), int(fo.value)

    def spchol_factor(self):
        self.spchol_factor_async()
        return self.spchol_factor_status()

    def spchol_solve(self, b):
        b = np.ascontiguousarray(b, np.float64)
        nrhs = 1 if b.ndim == 1 else b.shape[1]
        bb = b if b.ndim == 1 else np.asfortranarray(b)
        x = np.empty_like(bb)
        _check(self._L.spchol_solve(self._h, _vp(bb), _vp(x), nrhs, self.n))
        return x

    def spchol_solve_device(self, d_b: int, d_x: int, nrhs: int = 1, ld: int | None = None, stream: int | None = None):
        _check(self._L.spchol_solve_device(self._h, ctypes.c_void_p(d_b), ctypes.c_void_p(d_x), nrhs,
                                           self.n if ld is None else ld,
                                           ctypes.c_void_p(stream) if stream else None))

    def spchol_query(self, key):
        v = ctypes.c_int64()
        _check(self._L.spchol_query(self._h, Q[key] if isinstance(key, str) else key, ctypes.byref(v)))
        return int(v.value)

    def spchol_export_symbolic(self):
        q = self.spchol_query
        n, nf, ns = self.n, q("NFUND"), q("NSUPER")
        np_, rl, rlen = q("NPAIRS"), q("RELIND_LEN"), q("ROWS_LEN")
        d = dict(post=np.empty(n, np.int32), parent3=np.empty(n, np.int32), cc3=np.empty(n, np.int32),
                 ffirst=np.empty(nf + 1, np.int32), fgroup=np.empty(nf, np.int32),
                 perm_final=np.empty(n, np.int32), sfirst=np.empty(ns + 1, np.int32),
                 sparent=np.empty(ns, np.int32), rows_ptr=np.empty(ns + 1, np.int64),
                 rows=np.empty(rlen, np.int32), rel_ptr=np.empty(ns + 1, np.int64),
                 rel_anc=np.empty(np_, np.int32), rel_q0=np.empty(np_, np.int32),
                 rel_off=np.empty(np_ + 1, np.int64), relind=np.empty(rl, np.int32),
                 parent_final=np.empty(n, np.int32), cc_final=np.empty(n, np.int32),
                 level=np.empty(ns, np.int32))
        order = ["post", "parent3", "cc3", "ffirst", "fgroup", "perm_final", "sfirst", "sparent", "rows_ptr",
                 "rows", "rel_ptr", "rel_anc", "rel_q0", "rel_off", "relind", "parent_final", "cc_final", "level"]
        _check(self._L.spchol_export_symbolic(self._h, *[_vp(d[k]) for k in order]))
        return d

    def spchol_export_blocks(self):
        ns, nb = self.spchol_query("NSUPER"), self.spchol_query("NBLOCKS")
        d = dict(blk_ptr=np.empty(ns + 1, np.int64), blk_q=np.empty(nb, np.int32), blk_len=np.empty(nb, np.int32),
                 blk_anc=np.empty(nb, np.int32), blk_relind=np.empty(nb, np.int32))
        _check(self._L.spchol_export_blocks(self._h, *[_vp(d[k]) for k in ("blk_ptr", "blk_q", "blk_len", "blk_anc",
                                                                             "blk_relind")]))
        return d

    def spchol_export_panels(self, values=True):
        ns = self.spchol_query("NSUPER")
        off = np.empty(ns + 1, np.int64)
        ld = np.empty(ns, np.int32)
        pan = np.empty(self.spchol_query("PANEL_DOUBLES"), np.float64) if values else None
        _check(self._L.spchol_export_panels(self._h, _vp(off), _vp(ld), _vp(pan)))
        return off, ld, pan

    def spchol_export_panel(self, J):
        off, ld, _ = self.spchol_export_panels(values=False)
        k = np.diff(self.spchol_export_symbolic()["sfirst"])[J]
        out = np.empty(int(ld[J]) * int(k), np.float64)
        _check(self._L.spchol_export_panel(self._h, int(J), _vp(out)))
        return out.reshape(-1, int(ld[J])).T if out.size else out.reshape(0, 0)

    def spchol_export_diagonal(self):
        d = np.empty(self.n, np.float64)
        _check(self._L.spchol_export_diagonal(self._h, _vp(d)))
        return d

    def spchol_enable_kernel_timing(self, enable=True):
        _check(self._L.spchol_enable_kernel_timing(self._h, 1 if enable else 0))

    def spchol_kernel_stats(self, kind):
        n, ms, fl, by = ctypes.c_int64(), ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        k = KERNEL_KINDS[kind] if isinstance(kind, str) else kind
        _check(self._L.spchol_kernel_stats(self._h, k, ctypes.byref(n), ctypes.byref(ms), ctypes.byref(fl),
                                           ctypes.byref(by)))
        return dict(launches=int(n.value), ms=ms.value, flops=fl.value, bytes=by.value)

    def spchol_kernel_trace(self, cap=100000):
        cnt = ctypes.c_int64()
        kinds, levels = np.empty(cap, np.int32), np.empty(cap, np.int32)
        ntasks, ms = np.empty(cap, np.int32), np.empty(cap, np.float64)
        _check(self._L.spchol_kernel_trace(self._h, cap, ctypes.byref(cnt), _vp(kinds), _vp(levels), _vp(ntasks),
                                           _vp(ms)))
        c = min(cap, int(cnt.value))
        return dict(kinds=kinds[:c], levels=levels[:c], ntasks=ntasks[:c], ms=ms[:c])

    # ---- multi-GPU
    def spchol_dist_attach_nccl(self, unique_id: bytes):
        buf = ctypes.create_string_buffer(bytes(unique_id), 128)
        _check(self._L.spchol_dist_attach_nccl(self._h, buf))

    def spchol_export_mapping(self, with_top_owner=False):
        owner = np.empty(self.spchol_query("NSUPER"), np.int32)
        towner = np.empty(self.spchol_query("NSUPER"), np.int32)
        to, ts = ctypes.c_int64(), ctypes.c_int64()
        _check(self._L.spchol_export_mapping(self._h, _vp(owner), _vp(towner), ctypes.byref(to), ctypes.byref(ts)))
        if with_top_owner:
            return owner, towner, int(to.value), int(ts.value)
        return owner, int(to.value), int(ts.value)

    def spchol_dist_plan_flops(self):
        """(phase-A flops, per-level phase-C flops) of this rank's plan."""
        a = ctypes.c_double()
        lv = np.zeros(self.spchol_query("NLEVELS"), np.float64)
        _check(self._L.spchol_dist_plan_flops(self._h, ctypes.byref(a), _vp(lv)))
        return float(a.value), lv

    # ---- convenience (still only marshalling)
    factor = spchol_factor
    solve = spchol_solve
    query = spchol_query

    def factor_csc(self):
        """The computed L in the final numbering as CSC over the exact pattern (from the panels)."""
        sym = self.spchol_export_symbolic()
        off, ld, pan = self.spchol_export_panels()
        return sym, off, ld, pan


def spchol_dist_init(rank: int, world: int, unique_id: bytes | None = None):
    """Process-wide multi-GPU setup: later analyze calls with the default dist_world build this rank."""
    buf = ctypes.create_string_buffer(bytes(unique_id), 128) if unique_id is not None else None
    _check(lib().spchol_dist_init(int(rank), int(world), buf))


def spchol_dist_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().spchol_dist_nccl_unique_id(buf))
    return buf.raw


def analyze(n, colptr, rowidx, values=None, perm=None, **options) -> Solver:
    return Solver(n, colptr, rowidx, values, perm, **options)
