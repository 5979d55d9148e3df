"""Shared test helpers: compare the CUDA path's panels with the oracle (no method arithmetic here)."""
import math

import numpy as np

import gen


def panel_index_of_pattern(sym, off, ld, Lp, Li):
    """For every exact entry of L (CSC in final numbering) its index in the panel arena."""
    n = len(Lp) - 1
    sf, rp, rows = sym["sfirst"], sym["rows_ptr"], sym["rows"]
    ns = len(sf) - 1
    snode = np.repeat(np.arange(ns), np.diff(sf))
    col = np.repeat(np.arange(n), np.diff(Lp))
    J = snode[col]
    rowsJ = np.repeat(np.arange(ns), np.diff(rp))
    key_rows = rowsJ.astype(np.int64) * n + rows
    key = J.astype(np.int64) * n + Li
    idx = np.searchsorted(key_rows, key)
    assert np.all(key_rows[idx] == key), "exact nonzero outside its panel"
    q = idx - rp[J]
    c = col - sf[J]
    return off[J] + c * ld[J].astype(np.int64) + q


def lower_panel_mask(sym, off, ld, total):
    """Boolean mask of the panel arena: True on the stored lower part (row q >= column c, q < m)."""
    sf, rp = sym["sfirst"], sym["rows_ptr"]
    mask = np.zeros(total, bool)
    for J in range(len(sf) - 1):
        k = sf[J + 1] - sf[J]
        m = rp[J + 1] - rp[J]
        L = int(ld[J])
        blk = np.zeros((k, L), bool)
        qi = np.arange(L)
        for c in range(k):
            blk[c] = (qi >= c) & (qi < m)
        mask[off[J]:off[J] + k * L] = blk.ravel()     # panels need not be stored in supernode order
    return mask


inf_norm = gen.inf_norm
backward_error = gen.backward_error


def logdet_from_diag(diag):
    return 2.0 * math.fsum(np.log(diag).tolist())


def symmetric_csc(prob):
    """A (both triangles) as a scipy CSC matrix in the caller's numbering (verification only)."""
    import scipy.sparse as sps
    n = prob.n
    col = np.repeat(np.arange(n), np.diff(prob.colptr))
    Lw = sps.csc_matrix((prob.values, (prob.rowidx, col)), shape=(n, n))
    return (Lw + Lw.T - sps.diags(Lw.diagonal())).tocsc()


def llt_columns(sym, off, ld, pan, cols):
    """Columns `cols` (final numbering) of L L^T on and below the diagonal, computed from the exported
    panels: (L L^T)(i, j) = sum_{k <= j} L(i, k) L(j, k), where the k with L(j, k) != 0 are the
    columns of the supernodes K with j in rows(K) (padding entries are exactly 0).  Returns, per
    column j, (rows i >= j of rows(snode(j)), values)."""
    sf, rp, rows = sym["sfirst"], sym["rows_ptr"], sym["rows"]
    ns = len(sf) - 1
    owner = np.repeat(np.arange(ns), np.diff(rp))          # supernode of each rows[] entry
    out = {}
    for j in cols:
        hits = np.where(rows == j)[0]                       # every supernode K with j in rows(K)
        J = int(np.searchsorted(sf, j, side="right") - 1)
        rJ = rows[rp[J]:rp[J + 1]]
        tgt = rJ[rJ >= j]
        acc = np.zeros(len(tgt))
        for h in hits:
            K = int(owner[h])
            k, m, L = int(sf[K + 1] - sf[K]), int(rp[K + 1] - rp[K]), int(ld[K])
            ncol = min(k, j - int(sf[K]) + 1)               # columns k <= j
            P = pan[off[K]:off[K] + k * L].reshape(k, L)[:ncol]   # P[c, q] = L(rows(K)[q], sf[K] + c)
            qj = int(h - rp[K])                             # rows(K) ascends: rows >= j are q >= qj
            v = P[:, qj] @ P[:, qj:m]                       # sum over the columns of K
            rK = rows[rp[K] + qj:rp[K + 1]]
            idx = np.searchsorted(tgt, rK)
            assert np.all(idx < len(tgt)) and np.all(tgt[np.minimum(idx, len(tgt) - 1)] == rK), \
                "rows of K below j outside rows(snode(j)) (containment, P:172)"
            acc[idx] += v                                   # rows of one K are distinct
        out[int(j)] = (tgt, acc)
    return out


def cf_columns(prob, Afull, perm_final, cols):
    """Columns `cols` of C_f = P_f A P_f^T (final numbering), rows >= j, as dicts row -> value."""
    iperm = np.empty_like(perm_final)
    iperm[perm_final] = np.arange(len(perm_final))
    res = {}
    for j in cols:
        o = iperm[j]
        r = Afull.indices[Afull.indptr[o]:Afull.indptr[o + 1]]
        v = Afull.data[Afull.indptr[o]:Afull.indptr[o + 1]]
        fr = perm_final[r]
        keep = fr >= j
        res[int(j)] = dict(zip(fr[keep].tolist(), v[keep].tolist()))
    return res


def llt_sample_error(prob, sym, off, ld, pan, cols):
    """max |(L L^T)(i, j) - C_f(i, j)| / max |A| over every stored row i >= j of the sampled columns
    (an exact-result check, SURVEY §8(c) / S:348: independent of the oracle and of the kernels), and
    the number of entries compared."""
    Afull = symmetric_csc(prob)
    llt = llt_columns(sym, off, ld, pan, cols)
    cf = cf_columns(prob, Afull, sym["perm_final"], cols)
    worst, cnt = 0.0, 0
    for j, (rws, vals) in llt.items():
        ref = np.array([cf[j].get(int(r), 0.0) for r in rws])
        worst = max(worst, float(np.abs(vals - ref).max()))
        cnt += len(rws)
        # A's entries of column j outside the panel rows would be a structural error
        assert set(cf[j]).issubset(set(rws.tolist()))
    return worst / np.abs(prob.values).max(), cnt


def top_level_columns(sym, nlev=3, per_sn=4, seed=0):
    """A deterministic sample of columns of the supernodes in the top `nlev` levels (root first)."""
    lvl, sf = sym["level"], sym["sfirst"]
    top = np.where(lvl >= lvl.max() - nlev + 1)[0]
    rng = np.random.default_rng(seed)
    cols = []
    for J in top:
        k = int(sf[J + 1] - sf[J])
        cols += (int(sf[J]) + rng.choice(k, size=min(per_sn, k), replace=False)).tolist()
    return sorted(set(cols))
