"""ORACLE — test infrastructure only (see oracle/oracle.c header).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this package.  The product path (paper_2409_14009_b200) never imports it.

ctypes wrapper over oracle/liboracle.so (plain C, -O2 -ffp-contract=off).
Parity unpinned: nothing — every exported function is pinned by tests/test_oracle_*.py
(see DESIGN.md §Oracle pins).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

_I32 = ctypes.POINTER(ctypes.c_int32)
_I64 = ctypes.POINTER(ctypes.c_int64)
_F64 = ctypes.POINTER(ctypes.c_double)


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make -C {os.path.dirname(_HERE)} oracle`")
        L = ctypes.CDLL(path)
        L.orc_symbolic.restype = ctypes.c_void_p
        L.orc_symbolic.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                   ctypes.c_void_p, ctypes.c_double, ctypes.c_int, ctypes.c_int]
        L.orc_symbolic_pr.restype = ctypes.c_void_p
        L.orc_symbolic_pr.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                      ctypes.c_void_p, ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_int]
        L.orc_numeric.restype = ctypes.c_int
        L.orc_numeric.argtypes = [ctypes.c_void_p, _I64]
        L.orc_numeric_parallel.restype = ctypes.c_int
        L.orc_numeric_parallel.argtypes = [ctypes.c_void_p, ctypes.c_int, _I64]
        L.orc_solve.restype = ctypes.c_int
        L.orc_solve.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        L.orc_free.restype = None
        L.orc_free.argtypes = [ctypes.c_void_p]
        for nm, t in [("n", ctypes.c_int64), ("nnzL", ctypes.c_int64), ("flops", ctypes.c_double),
                      ("nfund", ctypes.c_int32), ("added", ctypes.c_int64), ("nmerges", ctypes.c_int32),
                      ("nsuper", ctypes.c_int32), ("npairs", ctypes.c_int64), ("nblocks", ctypes.c_int64)]:
            f = getattr(L, "orc_get_" + nm)
            f.restype = t
            f.argtypes = [ctypes.c_void_p]
        for nm, t in [("post", _I32), ("parent3", _I32), ("cc3", _I32), ("ffirst", _I32), ("fparent", _I32),
                      ("fgroup", _I32), ("merge_child", _I32), ("merge_parent", _I32), ("merge_cost", _I64),
                      ("perm_final", _I32), ("o7", _I32), ("sfirst", _I32), ("sparent", _I32),
                      ("rows_ptr", _I64), ("rows", _I32), ("rel_ptr", _I64), ("rel_anc", _I32),
                      ("rel_q0", _I32), ("rel_off", _I64), ("relind", _I32), ("parent_final", _I32),
                      ("cc_final", _I32), ("Lp", _I64), ("Li", _I32), ("Lx", _F64), ("blk_ptr", _I64),
                      ("blk_q", _I32), ("blk_len", _I32), ("blk_anc", _I32), ("blk_relind", _I32)]:
            f = getattr(L, "orc_ptr_" + nm)
            f.restype = t
            f.argtypes = [ctypes.c_void_p]
        _LIB = L
    return _LIB


def _vp(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


class OracleError(RuntimeError):
    pass


class Oracle:
    """Runs O1-O8 on construction (O7b partition refinement with pr=1); ``factor()`` runs O9,
    ``solve()`` O10."""

    def __init__(self, n, colptr, rowidx, values=None, perm=None, cap=0.25, rule=0, keep_L=True, pr=0):
        self._L = lib()
        self._keep = [np.ascontiguousarray(colptr, np.int64), np.ascontiguousarray(rowidx, np.int32),
                      None if values is None else np.ascontiguousarray(values, np.float64),
                      None if perm is None else np.ascontiguousarray(perm, np.int32)]
        cp, ri, vx, pm = self._keep
        self.n = int(n)
        h = self._L.orc_symbolic_pr(self.n, _vp(cp), _vp(ri), _vp(vx), _vp(pm), float(cap), int(rule), int(keep_L),
                                    int(pr))
        if not h:
            raise OracleError("oracle symbolic self-check failed")
        self._h = h
        self.factored = False

    @classmethod
    def from_problem(cls, prob, **kw):
        return cls(prob.n, prob.colptr, prob.rowidx, prob.values, prob.perm, **kw)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            self._L.orc_free(h)
            self._h = None

    def _get(self, nm):
        return getattr(self._L, "orc_get_" + nm)(self._h)

    def _arr(self, nm, count, dtype):
        if count == 0:
            return np.zeros(0, dtype)
        p = getattr(self._L, "orc_ptr_" + nm)(self._h)
        if not p:
            return None
        return np.ctypeslib.as_array(p, shape=(int(count),)).astype(dtype, copy=True)

    # scalar facts
    nnzL = property(lambda s: int(s._get("nnzL")))
    flops = property(lambda s: float(s._get("flops")))
    nfund = property(lambda s: int(s._get("nfund")))
    nsuper = property(lambda s: int(s._get("nsuper")))
    added = property(lambda s: int(s._get("added")))
    nmerges = property(lambda s: int(s._get("nmerges")))
    npairs = property(lambda s: int(s._get("npairs")))
    nblocks = property(lambda s: int(s._get("nblocks")))

    def symbolic(self):
        """All integer symbolic arrays (the bit-exact contract)."""
        n, nf, ns, npairs = self.n, self.nfund, self.nsuper, self.npairs
        d = dict(
            post=self._arr("post", n, np.int32), parent3=self._arr("parent3", n, np.int32),
            cc3=self._arr("cc3", n, np.int32), ffirst=self._arr("ffirst", nf + 1, np.int32),
            fparent=self._arr("fparent", nf, np.int32), fgroup=self._arr("fgroup", nf, np.int32),
            perm_final=self._arr("perm_final", n, np.int32), o7=self._arr("o7", n, np.int32),
            sfirst=self._arr("sfirst", ns + 1, np.int32), sparent=self._arr("sparent", ns, np.int32),
            rows_ptr=self._arr("rows_ptr", ns + 1, np.int64),
            rel_ptr=self._arr("rel_ptr", ns + 1, np.int64),
            rel_anc=self._arr("rel_anc", npairs, np.int32), rel_q0=self._arr("rel_q0", npairs, np.int32),
            rel_off=self._arr("rel_off", npairs + 1, np.int64),
            parent_final=self._arr("parent_final", n, np.int32), cc_final=self._arr("cc_final", n, np.int32),
        )
        d["rows"] = self._arr("rows", d["rows_ptr"][-1], np.int32)
        d["relind"] = self._arr("relind", d["rel_off"][-1], np.int32)
        nbk = self.nblocks
        d["blk_ptr"] = self._arr("blk_ptr", ns + 1, np.int64)
        for nmk in ("blk_q", "blk_len", "blk_anc", "blk_relind"):
            d[nmk] = self._arr(nmk, nbk, np.int32)
        nm = self.nmerges
        d["merges"] = list(zip(self._arr("merge_child", nm, np.int32).tolist(),
                               self._arr("merge_parent", nm, np.int32).tolist(),
                               self._arr("merge_cost", nm, np.int64).tolist()))
        return d

    def factor(self, threads=None):
        """O9.  threads=None: the serial build; threads=T: the level-parallel build on T threads
        (bit-identical L, the separately timed CPU baseline)."""
        fc = ctypes.c_int64(-1)
        if threads is None:
            rc = self._L.orc_numeric(self._h, ctypes.byref(fc))
        else:
            rc = self._L.orc_numeric_parallel(self._h, int(threads), ctypes.byref(fc))
        if rc == -3:
            return int(fc.value)
        if rc != 0:
            raise OracleError(f"orc_numeric rc={rc}")
        self.factored = True
        return -1

    def L_csc(self):
        """Exact factor of C_f = P_f A P_f^T: (Lp int64, Li int32, Lx float64 or None)."""
        Lp = self._arr("Lp", self.n + 1, np.int64)
        Li = self._arr("Li", Lp[-1], np.int32)
        Lx = self._arr("Lx", Lp[-1], np.float64) if self.factored else None
        return Lp, Li, Lx

    def solve(self, b):
        b = np.ascontiguousarray(b, np.float64)
        x = np.empty_like(b)
        rc = self._L.orc_solve(self._h, _vp(b), _vp(x))
        if rc != 0:
            raise OracleError(f"orc_solve rc={rc}")
        return x
