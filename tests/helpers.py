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
