"""Seeded synthetic inputs (shared by tests, oracle runs and the CUDA path).

Holds none of the method's arithmetic.
The grid/ND code is C (``gen/gen.c`` -> ``gen/libgen.so``) because the configs reach n = 4M.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

# id, stencil kind, grid, dof.  C1..C5 are BASELINE.json's configs; S* are parity-size
# members of the same families (the oracle factors them in seconds).
CONFIGS = {
    "C1": dict(cid=1, kind=5, grid=(30, 30, 1), dof=1, desc="2D 5-point Laplacian 30x30, ND"),
    "C2": dict(cid=2, kind=9, grid=(2000, 2000, 1), dof=1, desc="2D 9-point Laplacian 2000x2000, ND"),
    "C3": dict(cid=3, kind=7, grid=(64, 64, 64), dof=1, desc="3D 7-point Laplacian 64^3, ND"),
    "C4": dict(cid=4, kind=27, grid=(100, 100, 100), dof=1, desc="3D 27-point Laplacian 100^3, ND"),
    "C5": dict(cid=5, kind=27, grid=(70, 70, 70), dof=3, desc="3-dof 27-point elasticity-like 70^3, ND"),
    # parity-size members of the same families
    "S2": dict(cid=12, kind=9, grid=(120, 120, 1), dof=1, desc="2D 9-point 120x120, ND"),
    "S3": dict(cid=13, kind=7, grid=(24, 24, 24), dof=1, desc="3D 7-point 24^3, ND"),
    "S4": dict(cid=14, kind=27, grid=(20, 20, 20), dof=1, desc="3D 27-point 20^3, ND"),
    "S5": dict(cid=15, kind=27, grid=(12, 12, 12), dof=3, desc="3-dof 27-point 12^3, ND"),
    "T1": dict(cid=21, kind=5, grid=(7, 5, 1), dof=1, desc="2D 5-point 7x5 (ragged), ND"),
    "T2": dict(cid=22, kind=27, grid=(5, 4, 3), dof=3, desc="3-dof 27-point 5x4x3, ND"),
    "T3": dict(cid=23, kind=7, grid=(9, 7, 5), dof=1, desc="3D 7-point 9x7x5, ND"),
}
RHS_SEED_BASE = 0x2409140090000000


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "libgen.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make -C {os.path.dirname(_HERE)} gen`")
        L = ctypes.CDLL(path)
        L.gen_grid_csc.restype = ctypes.c_int64
        L.gen_grid_csc.argtypes = [ctypes.c_int] * 5 + [ctypes.c_void_p] * 3
        L.gen_nd_perm.restype = ctypes.c_int
        L.gen_nd_perm.argtypes = [ctypes.c_int] * 4 + [ctypes.c_void_p]
        L.gen_symv_lower.restype = None
        L.gen_symv_lower.argtypes = [ctypes.c_int64] + [ctypes.c_void_p] * 5
        L.gen_uniform.restype = None
        L.gen_uniform.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_double, ctypes.c_double, ctypes.c_void_p]
        _LIB = L
    return _LIB


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


@dataclass
class Problem:
    name: str
    n: int
    colptr: np.ndarray   # int64 [n+1]
    rowidx: np.ndarray   # int32 [nnz]
    values: np.ndarray   # float64 [nnz]
    perm: np.ndarray     # int32 [n], old -> new
    grid: tuple = ()
    dof: int = 1
    kind: int = 0

    @property
    def nnz(self):
        return int(self.colptr[-1])


def grid_matrix(kind, kx, ky, kz=1, dof=1):
    L = lib()
    n = kx * ky * kz * dof
    nnz = L.gen_grid_csc(kind, kx, ky, kz, dof, None, None, None)
    colptr = np.empty(n + 1, np.int64)
    rowidx = np.empty(nnz, np.int32)
    values = np.empty(nnz, np.float64)
    L.gen_grid_csc(kind, kx, ky, kz, dof, _p(colptr), _p(rowidx), _p(values))
    return n, colptr, rowidx, values


def nd_perm(kx, ky, kz=1, dof=1):
    perm = np.empty(kx * ky * kz * dof, np.int32)
    rc = lib().gen_nd_perm(kx, ky, kz, dof, _p(perm))
    if rc != 0:
        raise RuntimeError(f"gen_nd_perm failed ({rc})")
    return perm


def make(name: str) -> Problem:
    c = CONFIGS[name]
    kx, ky, kz = c["grid"]
    n, colptr, rowidx, values = grid_matrix(c["kind"], kx, ky, kz, c["dof"])
    return Problem(name, n, colptr, rowidx, values, nd_perm(kx, ky, kz, c["dof"]), (kx, ky, kz), c["dof"], c["kind"])


def make_grid(kind, kx, ky, kz=1, dof=1, name=None) -> Problem:
    n, colptr, rowidx, values = grid_matrix(kind, kx, ky, kz, dof)
    return Problem(name or f"g{kind}_{kx}x{ky}x{kz}x{dof}", n, colptr, rowidx, values,
                   nd_perm(kx, ky, kz, dof), (kx, ky, kz), dof, kind)


def uniform(seed: int, n: int, lo=-1.0, hi=1.0):
    out = np.empty(n, np.float64)
    lib().gen_uniform(ctypes.c_uint64(seed & (2**64 - 1)), n, lo, hi, _p(out))
    return out


def symv(prob_or_n, colptr=None, rowidx=None, values=None, x=None):
    """y = A x for the symmetric A stored as its lower triangle."""
    if isinstance(prob_or_n, Problem):
        n, colptr, rowidx, values = prob_or_n.n, prob_or_n.colptr, prob_or_n.rowidx, prob_or_n.values
    else:
        n = prob_or_n
    x = np.ascontiguousarray(x, np.float64)
    y = np.empty(n, np.float64)
    lib().gen_symv_lower(n, _p(colptr), _p(rowidx), _p(values), _p(x), _p(y))
    return y


def rhs(prob: Problem):
    """x*_i ~ U[-1,1) from splitmix64(seed = 0x2409140090000000 + config id); b = A x*."""
    cid = CONFIGS[prob.name]["cid"] if prob.name in CONFIGS else 0
    xstar = uniform(RHS_SEED_BASE + cid, prob.n)
    return xstar, symv(prob, x=xstar)


# ---- random tiny SPD corpus (SURVEY §8(c) "Random tiny corpus") ----
def _splitmix_stream(seed):
    s = seed & (2**64 - 1)
    M = 2**64 - 1
    while True:
        s = (s + 0x9E3779B97F4A7C15) & M
        z = s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        yield z ^ (z >> 31)


def random_spd(trial: int, n: int | None = None, p: float | None = None, shuffle: bool | None = None):
    """Strictly diagonally dominant random SPD pattern; returns a Problem in lower CSC."""
    g = _splitmix_stream(trial)
    u = lambda: (next(g) >> 11) * (1.0 / 9007199254740992.0)
    if n is None:
        n = 1 + int(u() * 64)
    if p is None:
        p = (0.05, 0.15, 0.4)[int(u() * 3)]
    if shuffle is None:
        shuffle = u() < 0.5
    dense = np.zeros((n, n))
    for j in range(n):
        for i in range(j + 1, n):
            if u() < p:
                dense[i, j] = -(0.1 + 0.9 * u())
    full = dense + dense.T
    diag = np.abs(full).sum(axis=1) + 1.0
    np.fill_diagonal(dense, diag)
    perm = np.arange(n, dtype=np.int32)
    if shuffle:
        for i in range(n - 1, 0, -1):  # Fisher-Yates
            k = int(u() * (i + 1))
            perm[i], perm[k] = perm[k], perm[i]
    return from_dense_lower(dense, perm, name=f"rand{trial}")


def from_dense_lower(dense, perm=None, name="dense"):
    n = dense.shape[0]
    colptr = np.zeros(n + 1, np.int64)
    rows, vals = [], []
    for j in range(n):
        idx = [j] + [i for i in range(j + 1, n) if dense[i, j] != 0.0]
        rows.extend(idx)
        vals.extend(dense[i, j] for i in idx)
        colptr[j + 1] = len(rows)
    if perm is None:
        perm = np.arange(n, dtype=np.int32)
    return Problem(name, n, colptr, np.array(rows, np.int32), np.array(vals, np.float64),
                   np.asarray(perm, np.int32))


def to_dense(prob: Problem):
    A = np.zeros((prob.n, prob.n))
    for j in range(prob.n):
        for p in range(prob.colptr[j], prob.colptr[j + 1]):
            i = prob.rowidx[p]
            A[i, j] = prob.values[p]
            A[j, i] = prob.values[p]
    return A


def leading_submatrix(prob: Problem, ns: int) -> Problem:
    """The leading ns x ns principal submatrix of P A P^T (P = prob.perm), in that order, identity perm.

    Used as the bounded CPU-baseline sample: in nested-dissection order the leading block is a
    union of whole ND subtrees, so its factor is exactly the leading block of the full factor.
    """
    inv = np.argsort(prob.perm)
    newidx = np.full(prob.n, -1, np.int64)
    newidx[inv[:ns]] = np.arange(ns)
    colid = np.repeat(np.arange(prob.n), np.diff(prob.colptr))
    r, c = newidx[prob.rowidx], newidx[colid]
    keep = (r >= 0) & (c >= 0)
    r, c, v = r[keep], c[keep], prob.values[keep]
    lo, hi = np.minimum(r, c), np.maximum(r, c)
    order = np.lexsort((hi, lo))
    lo, hi, v = lo[order], hi[order], v[order]
    colptr = np.zeros(ns + 1, np.int64)
    np.add.at(colptr, lo + 1, 1)
    return Problem(f"{prob.name}[:{ns}]", ns, np.cumsum(colptr), hi.astype(np.int32), v.astype(np.float64),
                   np.arange(ns, dtype=np.int32), prob.grid, prob.dof, prob.kind)


def inf_norm(prob: Problem) -> float:
    """||A||_inf of the symmetric A stored as its lower triangle."""
    rowsum = np.zeros(prob.n)
    cols = np.repeat(np.arange(prob.n), np.diff(prob.colptr))
    np.add.at(rowsum, prob.rowidx, np.abs(prob.values))
    off = prob.rowidx != cols
    np.add.at(rowsum, cols[off], np.abs(prob.values[off]))
    return float(rowsum.max())


def backward_error(prob: Problem, x, b) -> float:
    """Normwise backward error ||A x - b||_inf / (||A||_inf ||x||_inf) (verification only)."""
    r = symv(prob, x=x) - b
    return float(np.abs(r).max() / (inf_norm(prob) * np.abs(x).max()))
