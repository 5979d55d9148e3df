// spchol_analyze's symbolic phase: the product's fast path (host, integer only).
//
// Algorithms (all O(nnz) or O(nnz log) — the configs reach n = 4M, nnz(L) = 2.3e9):
//   permutation of the pattern by counting sorts            (perm is an input)
//   elimination tree: Liu's algorithm with path compression  (FIND/UNION P:27,68)
//   postorder from subtree sizes (children ascending)        (reading R6)
//   column counts: Gilbert-Ng-Peyton with lca/prevleaf       (macros lca/prevlf/fchild P:21-52)
//   fundamental supernodes [LNP93]                           (reading R1)
//   greedy child-parent merging with an indexed heap         (readings R3-R6)
//   final permutation = postorder of the merged tree         (reading R6)
//   optional partition refinement inside the supernodes       (reading R14)
//   rows(J) by supernodal symbolic factorization on the merged partition
//   relind(J,P) via indmap                                    (indmap P:38-39)
//   level sets (heights) of the merged supernodal tree      (north_star: level-set scheduling)
// This file shares no code with oracle/ (the CPU test oracle); both follow the paper.
#include <algorithm>
#include <cstring>
#include <numeric>

#include "spchol.h"
#include "symbolic.h"

namespace spchol {
namespace {

// Lower-triangular pattern of Q M Q^T from a lower CSC M (q[old] = new), rows ascending.
// Also returns the row-wise (CSR) form and, optionally, the source entry of every output entry.
struct Pat {
  std::vector<int64_t> cp;  // CSC column pointers
  std::vector<int32_t> ci;  // CSC row indices (ascending per column)
  std::vector<int64_t> src; // CSC: source entry index (optional)
  std::vector<int64_t> rp;  // CSR row pointers
  std::vector<int32_t> rj;  // CSR column indices (ascending per row)
};

void permute_pattern(int64_t n, const int64_t* colptr, const int32_t* rowidx, const int32_t* q,
                     bool want_src, bool want_csr, Pat& out) {
  const int64_t nnz = colptr[n];
  // pass 1: bucket entries by new column
  std::vector<int64_t> cnt(n + 1, 0);
  for (int64_t j = 0; j < n; ++j)
    for (int64_t p = colptr[j]; p < colptr[j + 1]; ++p) {
      int32_t a = q[rowidx[p]], b = q[j];
      cnt[(a < b ? a : b) + 1]++;
    }
  for (int64_t j = 0; j < n; ++j) cnt[j + 1] += cnt[j];
  std::vector<int64_t> byc(nnz);
  {
    std::vector<int64_t> nx(cnt.begin(), cnt.end() - 1);
    for (int64_t j = 0; j < n; ++j)
      for (int64_t p = colptr[j]; p < colptr[j + 1]; ++p) {
        int32_t a = q[rowidx[p]], b = q[j];
        byc[nx[a < b ? a : b]++] = p;
      }
  }
  // we need each entry's original column; build an entry -> original column map lazily
  std::vector<int32_t> ecol(nnz);
  for (int64_t j = 0; j < n; ++j)
    for (int64_t p = colptr[j]; p < colptr[j + 1]; ++p) ecol[p] = (int32_t)j;
  auto newrow = [&](int64_t p) { int32_t a = q[rowidx[p]], b = q[ecol[p]]; return a < b ? b : a; };
  auto newcol = [&](int64_t p) { int32_t a = q[rowidx[p]], b = q[ecol[p]]; return a < b ? a : b; };
  // pass 2: columns ascending -> bucket by row (each row's list gets columns ascending)
  std::vector<int64_t> rcnt(n + 1, 0);
  for (int64_t p = 0; p < nnz; ++p) rcnt[newrow(p) + 1]++;
  for (int64_t i = 0; i < n; ++i) rcnt[i + 1] += rcnt[i];
  std::vector<int64_t> byr(nnz);
  {
    std::vector<int64_t> nx(rcnt.begin(), rcnt.end() - 1);
    for (int64_t t = 0; t < nnz; ++t) { int64_t p = byc[t]; byr[nx[newrow(p)]++] = p; }
  }
  if (want_csr) {
    out.rp = rcnt;
    out.rj.resize(nnz);
    for (int64_t t = 0; t < nnz; ++t) out.rj[t] = newcol(byr[t]);
  }
  // pass 3: rows ascending -> bucket by column (each column's rows ascending)
  out.cp = cnt;
  out.ci.resize(nnz);
  if (want_src) out.src.resize(nnz);
  std::vector<int64_t> nx(cnt.begin(), cnt.end() - 1);
  for (int64_t t = 0; t < nnz; ++t) {
    int64_t p = byr[t];
    int64_t d = nx[newcol(p)]++;
    out.ci[d] = newrow(p);
    if (want_src) out.src[d] = p;
  }
}

// Indexed binary min-heap on (key, id).
struct IHeap {
  std::vector<int32_t> h, pos;
  std::vector<int64_t> key;
  explicit IHeap(int32_t n) : pos(n, -1), key(n, 0) {}
  bool lt(int32_t a, int32_t b) const { return key[a] < key[b] || (key[a] == key[b] && a < b); }
  void sw(size_t i, size_t j) { std::swap(h[i], h[j]); pos[h[i]] = (int32_t)i; pos[h[j]] = (int32_t)j; }
  void up(size_t i) { while (i > 0) { size_t p = (i - 1) / 2; if (!lt(h[i], h[p])) break; sw(i, p); i = p; } }
  void down(size_t i) {
    for (;;) {
      size_t l = 2 * i + 1, r = l + 1, m = i;
      if (l < h.size() && lt(h[l], h[m])) m = l;
      if (r < h.size() && lt(h[r], h[m])) m = r;
      if (m == i) return;
      sw(i, m); i = m;
    }
  }
  void set(int32_t id, int64_t k) {
    if (pos[id] < 0) { key[id] = k; pos[id] = (int32_t)h.size(); h.push_back(id); up(h.size() - 1); return; }
    int64_t old = key[id]; key[id] = k;
    if (k < old) up((size_t)pos[id]); else down((size_t)pos[id]);
  }
  void remove(int32_t id) {
    int32_t i = pos[id];
    if (i < 0) return;
    size_t last = h.size() - 1;
    if ((size_t)i != last) sw((size_t)i, last);
    h.pop_back(); pos[id] = -1;
    if ((size_t)i < h.size()) { down((size_t)i); up((size_t)i); }
  }
  bool empty() const { return h.empty(); }
  int32_t top() const { return h[0]; }
};

}  // namespace

int analyze_symbolic(int64_t n, const int64_t* colptr, const int32_t* rowidx, const int32_t* perm_in,
                     double cap, int pr, Symbolic& S, std::string& err) {
  if (n < 0) { err = "n < 0"; return SPCHOL_ERR_DIMENSION; }
  if (n >= INT32_MAX) { err = "n must be < 2^31"; return SPCHOL_ERR_DIMENSION; }
  if (!colptr || (n > 0 && !rowidx)) { err = "NULL pattern arrays"; return SPCHOL_ERR_VALIDATION; }
  // ---- validate the CSC contract
  if (colptr[0] != 0) { err = "colptr[0] != 0"; return SPCHOL_ERR_VALIDATION; }
  for (int64_t j = 0; j < n; ++j) {
    if (colptr[j + 1] <= colptr[j]) { err = "column " + std::to_string(j) + " is empty (diagonal must be stored)"; return SPCHOL_ERR_VALIDATION; }
    if (rowidx[colptr[j]] != j) { err = "column " + std::to_string(j) + ": first entry is not the diagonal"; return SPCHOL_ERR_VALIDATION; }
    for (int64_t p = colptr[j] + 1; p < colptr[j + 1]; ++p)
      if (rowidx[p] <= rowidx[p - 1] || rowidx[p] >= n) { err = "column " + std::to_string(j) + ": rows not strictly increasing within [j,n)"; return SPCHOL_ERR_VALIDATION; }
  }
  S.n = n; S.nnzA = colptr[n];
  std::vector<int32_t> perm(n);
  if (perm_in) {
    std::vector<char> seen(n, 0);
    for (int64_t i = 0; i < n; ++i) {
      int32_t v = perm_in[i];
      if (v < 0 || v >= n || seen[v]) { err = "perm is not a bijection of [0,n)"; return SPCHOL_ERR_VALIDATION; }
      seen[v] = 1; perm[i] = v;
    }
  } else {
    std::iota(perm.begin(), perm.end(), 0);
  }
  // ---- permute: C = P A P^T (pattern, row form needed by Liu's algorithm)
  Pat C;
  permute_pattern(n, colptr, rowidx, perm.data(), false, true, C);
  // ---- elimination tree, Liu's algorithm with path compression (virtual ancestors)
  std::vector<int32_t> parent(n, -1), anc(n, -1);
  for (int64_t j = 0; j < n; ++j) {
    for (int64_t p = C.rp[j]; p < C.rp[j + 1]; ++p) {
      int32_t r = C.rj[p];
      if (r >= j) continue;
      while (anc[r] != -1 && anc[r] != j) { int32_t nx = anc[r]; anc[r] = (int32_t)j; r = nx; }
      if (anc[r] == -1) { anc[r] = (int32_t)j; parent[r] = (int32_t)j; }
    }
  }
  std::vector<int32_t>().swap(anc);
  // ---- postorder from subtree sizes: children ascending, roots ascending
  std::vector<int32_t> ipost(n);
  {
    std::vector<int64_t> size(n, 1);
    for (int64_t j = 0; j < n; ++j) if (parent[j] != -1) size[parent[j]] += size[j];
    // children lists ascending (CSR by parent)
    std::vector<int64_t> kp(n + 1, 0);
    for (int64_t j = 0; j < n; ++j) if (parent[j] != -1) kp[parent[j] + 1]++;
    for (int64_t j = 0; j < n; ++j) kp[j + 1] += kp[j];
    std::vector<int32_t> kids(kp[n]);
    { std::vector<int64_t> nx(kp.begin(), kp.end() - 1);
      for (int64_t j = 0; j < n; ++j) if (parent[j] != -1) kids[nx[parent[j]]++] = (int32_t)j; }
    std::vector<int64_t> start(n, 0);
    int64_t cur = 0;
    for (int64_t r = 0; r < n; ++r) if (parent[r] == -1) { start[r] = cur; cur += size[r]; }
    for (int64_t v = n - 1; v >= 0; --v) {  // parents (larger index) before children
      int64_t c0 = start[v];
      for (int64_t p = kp[v]; p < kp[v + 1]; ++p) { start[kids[p]] = c0; c0 += size[kids[p]]; }
      ipost[v] = (int32_t)(start[v] + size[v] - 1);
    }
  }
  S.post.assign(n, 0);
  for (int64_t j = 0; j < n; ++j) S.post[ipost[j]] = (int32_t)j;
  S.parent3.assign(n, -1);
  for (int64_t j = 0; j < n; ++j) S.parent3[ipost[j]] = parent[j] == -1 ? -1 : ipost[parent[j]];
  std::vector<int32_t>().swap(parent);
  // ---- C3 = post-relabelled C (lower CSC); composite q = ipost o perm applied to A
  std::vector<int32_t> q3(n);
  for (int64_t i = 0; i < n; ++i) q3[i] = ipost[perm[i]];
  Pat C3;
  permute_pattern(n, colptr, rowidx, q3.data(), false, false, C3);
  { Pat tmp; std::swap(C, tmp); }
  // ---- column counts: Gilbert-Ng-Peyton (skeleton leaves, lca by path-compressed ancestors)
  const std::vector<int32_t>& par3 = S.parent3;
  S.cc3.assign(n, 0);
  {
    std::vector<int64_t> size(n, 1);
    for (int64_t j = 0; j < n; ++j) if (par3[j] != -1) size[par3[j]] += size[j];
    std::vector<int32_t> first(n), maxfirst(n, -1), prevleaf(n, -1), ancestor(n);
    std::vector<int64_t> delta(n, 0);
    for (int64_t j = 0; j < n; ++j) { first[j] = (int32_t)(j - size[j] + 1); ancestor[j] = (int32_t)j; delta[j] = size[j] == 1 ? 1 : 0; }
    for (int64_t j = 0; j < n; ++j) {
      if (par3[j] != -1) delta[par3[j]]--;
      for (int64_t p = C3.cp[j]; p < C3.cp[j + 1]; ++p) {
        int32_t i = C3.ci[p];
        if (i <= j || first[j] <= maxfirst[i]) continue;   // j is not a leaf of row subtree i
        maxfirst[i] = first[j];
        int32_t jprev = prevleaf[i];
        prevleaf[i] = (int32_t)j;
        delta[j]++;
        if (jprev != -1) {                                  // subsequent leaf: subtract at lca
          int32_t qq = jprev;
          while (qq != ancestor[qq]) qq = ancestor[qq];
          for (int32_t s = jprev, sp; s != qq; s = sp) { sp = ancestor[s]; ancestor[s] = qq; }
          delta[qq]--;
        }
      }
      if (par3[j] != -1) ancestor[j] = par3[j];
    }
    for (int64_t j = 0; j < n; ++j) if (par3[j] != -1) delta[par3[j]] += delta[j];
    for (int64_t j = 0; j < n; ++j) S.cc3[j] = (int32_t)delta[j];
  }
  S.nnzL = 0; S.flops_exact = 0.0;
  for (int64_t j = 0; j < n; ++j) { S.nnzL += S.cc3[j]; S.flops_exact += (double)S.cc3[j] * (double)S.cc3[j]; }
  // ---- fundamental supernodes (LNP93)
  std::vector<int32_t> nchild(n, 0), fsn(n);
  for (int64_t j = 0; j < n; ++j) if (par3[j] != -1) nchild[par3[j]]++;
  S.ffirst.clear();
  for (int64_t j = 0; j < n; ++j) {
    bool join = j > 0 && par3[j - 1] == j && S.cc3[j - 1] == S.cc3[j] + 1 && nchild[j] == 1;
    if (!join) S.ffirst.push_back((int32_t)j);
    fsn[j] = (int32_t)S.ffirst.size() - 1;
  }
  const int32_t nf = (int32_t)S.ffirst.size();
  S.ffirst.push_back((int32_t)n);
  S.fparent.assign(nf, -1);
  for (int32_t f = 0; f < nf; ++f) {
    int32_t last = S.ffirst[f + 1] - 1;
    S.fparent[f] = par3[last] == -1 ? -1 : fsn[par3[last]];
  }
  // ---- greedy merging: min (cost, child id), cost = k_J (k_J + m_P - m_J)
  std::vector<int64_t> gk(nf), gm(nf);
  std::vector<int32_t> gpar(S.fparent), into(nf, -1);
  std::vector<std::vector<int32_t>> gkids(nf);
  for (int32_t f = 0; f < nf; ++f) {
    gk[f] = S.ffirst[f + 1] - S.ffirst[f];
    gm[f] = S.cc3[S.ffirst[f]];
    if (gpar[f] != -1) gkids[gpar[f]].push_back(f);
  }
  S.added = 0; S.nmerges = 0;
  if (cap >= 0.0) {
    const double budget = cap * (double)S.nnzL;
    IHeap H(nf);
    auto cost = [&](int32_t J) { return gk[J] * (gk[J] + gm[gpar[J]] - gm[J]); };
    for (int32_t f = 0; f < nf; ++f) if (gpar[f] != -1) H.set(f, cost(f));
    while (!H.empty()) {
      int32_t J = H.top();
      int64_t c = H.key[J];
      if ((double)(S.added + c) > budget) break;   // never exceed (R4); costs only grow
      H.remove(J);
      int32_t P = gpar[J];
      S.added += c; S.nmerges++;
      gm[P] = gk[J] + gm[P];
      gk[P] = gk[J] + gk[P];
      into[J] = P;
      for (int32_t ch : gkids[J]) { gpar[ch] = P; gkids[P].push_back(ch); }
      std::vector<int32_t>().swap(gkids[J]);
      auto& kp = gkids[P];
      kp.erase(std::remove_if(kp.begin(), kp.end(), [&](int32_t x) { return into[x] != -1 || gpar[x] != P; }), kp.end());
      for (int32_t ch : kp) H.set(ch, cost(ch));
      if (gpar[P] != -1) H.set(P, cost(P));
    }
  }
  S.fgroup.assign(nf, 0);
  for (int32_t f = nf - 1; f >= 0; --f) S.fgroup[f] = into[f] == -1 ? f : S.fgroup[into[f]];  // into[f] > f
  // ---- final permutation: postorder of the merged tree, children by smallest column (R6)
  std::vector<int32_t> o7(n);
  std::vector<int32_t> groups;  // alive group ids
  for (int32_t f = 0; f < nf; ++f) if (into[f] == -1) groups.push_back(f);
  std::vector<int32_t> gmin(nf, INT32_MAX);
  std::vector<int64_t> gcols(nf, 0);
  for (int32_t f = 0; f < nf; ++f) {
    int32_t g = S.fgroup[f];
    gmin[g] = std::min(gmin[g], S.ffirst[f]);
    gcols[g] += S.ffirst[f + 1] - S.ffirst[f];
  }
  std::vector<int64_t> gsize(nf, 0), gstart(nf, 0);
  for (int32_t g : groups) gsize[g] = gcols[g];
  for (int32_t g : groups) if (gpar[g] != -1) gsize[gpar[g]] += gsize[g];  // ascending ids: kids first
  auto bymin = [&](int32_t a, int32_t b) { return gmin[a] < gmin[b]; };
  {
    std::vector<int32_t> roots;
    for (int32_t g : groups) if (gpar[g] == -1) roots.push_back(g);
    std::sort(roots.begin(), roots.end(), bymin);
    int64_t cur = 0;
    for (int32_t r : roots) { gstart[r] = cur; cur += gsize[r]; }
    for (auto it = groups.rbegin(); it != groups.rend(); ++it) {
      int32_t g = *it;
      auto& kd = gkids[g];
      std::sort(kd.begin(), kd.end(), bymin);
      int64_t c0 = gstart[g];
      for (int32_t ch : kd) { gstart[ch] = c0; c0 += gsize[ch]; }
    }
  }
  {
    std::vector<int64_t> nxt(nf);
    for (int32_t g : groups) nxt[g] = gstart[g] + gsize[g] - gcols[g];
    for (int64_t j = 0; j < n; ++j) o7[j] = (int32_t)(nxt[S.fgroup[fsn[j]]]++);  // ascending O3 inside
  }
  // supernodes in final order
  std::vector<int32_t> order(groups);
  std::sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return gstart[a] + gsize[a] < gstart[b] + gsize[b]; });
  const int32_t ns = (int32_t)order.size();
  S.nsuper = ns;
  std::vector<int32_t> sid(nf, -1);
  for (int32_t s = 0; s < ns; ++s) sid[order[s]] = s;
  S.sfirst.assign(ns + 1, 0);
  S.sparent.assign(ns, -1);
  std::vector<int64_t> mexp(ns);
  for (int32_t s = 0; s < ns; ++s) {
    int32_t g = order[s];
    S.sfirst[s] = (int32_t)(gstart[g] + gsize[g] - gcols[g]);
    S.sparent[s] = gpar[g] == -1 ? -1 : sid[gpar[g]];
    mexp[s] = gm[g];
  }
  S.sfirst[ns] = (int32_t)n;
  S.snode.assign(n, 0);
  for (int32_t s = 0; s < ns; ++s) for (int32_t c = S.sfirst[s]; c < S.sfirst[s + 1]; ++c) S.snode[c] = s;
  S.perm_final.assign(n, 0); S.iperm_final.assign(n, 0);
  for (int64_t i = 0; i < n; ++i) { S.perm_final[i] = o7[ipost[perm[i]]]; S.iperm_final[S.perm_final[i]] = (int32_t)i; }
  S.parent_final.assign(n, -1); S.cc_final.assign(n, 0);
  for (int64_t j = 0; j < n; ++j) {
    S.parent_final[o7[j]] = par3[j] == -1 ? -1 : o7[par3[j]];
    S.cc_final[o7[j]] = S.cc3[j];
  }
  { Pat tmp; std::swap(C3, tmp); }
  // ---- C_f pattern (+ source entries for the A -> panel map); supernodal symbolic for rows(J)
  Pat Cf;
  permute_pattern(n, colptr, rowidx, S.perm_final.data(), true, false, Cf);
  std::vector<std::vector<int32_t>> skids(ns);
  for (int32_t s = 0; s < ns; ++s) if (S.sparent[s] != -1) skids[S.sparent[s]].push_back(s);
  S.rows_ptr.assign(ns + 1, 0);
  for (int32_t s = 0; s < ns; ++s) S.rows_ptr[s + 1] = S.rows_ptr[s] + mexp[s];
  S.rows.assign(S.rows_ptr[ns], 0);
  {
    std::vector<int32_t> mark(n, -1), extra;
    for (int32_t s = 0; s < ns; ++s) {
      int32_t f = S.sfirst[s], l = S.sfirst[s + 1] - 1;
      extra.clear();
      for (int32_t j = f; j <= l; ++j)
        for (int64_t p = Cf.cp[j]; p < Cf.cp[j + 1]; ++p) {
          int32_t i = Cf.ci[p];
          if (i > l && mark[i] != s) { mark[i] = s; extra.push_back(i); }
        }
      for (int32_t t : skids[s]) {
        int64_t kt = S.sfirst[t + 1] - S.sfirst[t];
        for (int64_t p = S.rows_ptr[t] + kt; p < S.rows_ptr[t + 1]; ++p) {
          int32_t i = S.rows[p];
          if (i > l && mark[i] != s) { mark[i] = s; extra.push_back(i); }
        }
      }
      std::sort(extra.begin(), extra.end());
      int64_t k = l - f + 1;
      if (k + (int64_t)extra.size() != mexp[s]) {
        err = "internal: supernode row count mismatch";
        return SPCHOL_ERR_VALIDATION;
      }
      int64_t w = S.rows_ptr[s];
      for (int32_t c = f; c <= l; ++c) S.rows[w++] = c;
      for (int32_t i : extra) S.rows[w++] = i;
    }
  }
  // ---- partition refinement (reading R14): per supernode P, the ordered partition of cols(P) is
  // refined by S_J = R_J n cols(P), J ascending, each touched part split stably into (in S, not in
  // S).  Parts are position ranges [pstart, pend); only the parts S_J touches are visited.
  if (pr) {
    std::vector<int32_t> ord(n), where(n), pstart(n), pend(n), tmp(n);
    std::vector<char> inS(n, 0), touched(n, 0);
    for (int64_t i = 0; i < n; ++i) { ord[i] = (int32_t)i; where[i] = (int32_t)i; }
    for (int32_t P = 0; P < ns; ++P)
      for (int32_t i = S.sfirst[P]; i < S.sfirst[P + 1]; ++i) { pstart[i] = S.sfirst[P]; pend[i] = S.sfirst[P + 1]; }
    std::vector<int32_t> parts;
    for (int32_t J = 0; J < ns; ++J) {
      const int64_t k = S.sfirst[J + 1] - S.sfirst[J];
      const int32_t* r = S.rows.data() + S.rows_ptr[J];
      const int64_t m = S.rows_ptr[J + 1] - S.rows_ptr[J];
      for (int64_t q = k; q < m;) {
        const int32_t P = S.snode[r[q]];
        int64_t q1 = q;
        parts.clear();
        for (; q1 < m && S.snode[r[q1]] == P; ++q1) {
          inS[r[q1]] = 1;
          const int32_t a = pstart[where[r[q1]]];
          if (!touched[a]) { touched[a] = 1; parts.push_back(a); }
        }
        for (int32_t a : parts) {
          touched[a] = 0;
          const int32_t e = pend[a];
          int32_t w = a;
          for (int32_t i = a; i < e; ++i) if (inS[ord[i]]) tmp[w++] = ord[i];
          const int32_t mid = w;
          for (int32_t i = a; i < e; ++i) if (!inS[ord[i]]) tmp[w++] = ord[i];
          for (int32_t i = a; i < e; ++i) { ord[i] = tmp[i]; where[ord[i]] = i; }
          if (mid < e) {   // both halves nonempty (mid > a: the part held an element of S)
            for (int32_t i = a; i < mid; ++i) pend[i] = mid;
            for (int32_t i = mid; i < e; ++i) pstart[i] = mid;
          }
        }
        for (int64_t x = q; x < q1; ++x) inS[r[x]] = 0;
        q = q1;
      }
    }
    // relabel: newlab = position; rows(J) re-sorted; P_f and the A -> C_f map recomputed
    std::vector<int32_t>& newlab = where;
    for (int64_t x = 0; x < S.rows_ptr[ns]; ++x) S.rows[x] = newlab[S.rows[x]];
    for (int32_t sn = 0; sn < ns; ++sn) std::sort(S.rows.begin() + S.rows_ptr[sn], S.rows.begin() + S.rows_ptr[sn + 1]);
    for (int64_t i = 0; i < n; ++i) { S.perm_final[i] = newlab[S.perm_final[i]]; S.iperm_final[S.perm_final[i]] = (int32_t)i; }
    { Pat tmp2; std::swap(Cf, tmp2); }
    permute_pattern(n, colptr, rowidx, S.perm_final.data(), true, true, Cf);
    // the exact factor's structure in the refined order: Liu's etree, then column counts by
    // walking every row subtree (row i: from each k with C_f(i,k) != 0 up the etree to i)
    std::vector<int32_t> anc(n, -1);
    for (int64_t j = 0; j < n; ++j) {
      S.parent_final[j] = -1;
      for (int64_t p = Cf.rp[j]; p < Cf.rp[j + 1]; ++p) {
        int32_t rr = Cf.rj[p];
        if (rr >= j) continue;
        while (anc[rr] != -1 && anc[rr] != j) { int32_t nx = anc[rr]; anc[rr] = (int32_t)j; rr = nx; }
        if (anc[rr] == -1) { anc[rr] = (int32_t)j; S.parent_final[rr] = (int32_t)j; }
      }
    }
    std::vector<int32_t> mark(n, -1);
    for (int64_t j = 0; j < n; ++j) S.cc_final[j] = 1;
    for (int64_t i = 0; i < n; ++i) {
      mark[i] = (int32_t)i;
      for (int64_t p = Cf.rp[i]; p < Cf.rp[i + 1]; ++p)
        for (int32_t kk = Cf.rj[p]; kk >= 0 && mark[kk] != i; kk = S.parent_final[kk]) { mark[kk] = (int32_t)i; S.cc_final[kk]++; }
    }
    S.nnzL = 0; S.flops_exact = 0.0;
    for (int64_t j = 0; j < n; ++j) { S.nnzL += S.cc_final[j]; S.flops_exact += (double)S.cc_final[j] * (double)S.cc_final[j]; }
  }
  // ---- levels (height from the leaves)
  S.level.assign(ns, 0);
  for (int32_t s = 0; s < ns; ++s)
    if (S.sparent[s] != -1) S.level[S.sparent[s]] = std::max(S.level[S.sparent[s]], S.level[s] + 1);
  S.nlevels = 0;
  for (int32_t s = 0; s < ns; ++s) S.nlevels = std::max(S.nlevels, S.level[s] + 1);
  // ---- relind via indmap, pairs grouped by ancestor
  {
    std::vector<int32_t> pj, pp, pq;  // pair: J, P, q0
    S.rel_ptr.assign(ns + 1, 0);
    for (int32_t J = 0; J < ns; ++J) {
      int64_t k = S.sfirst[J + 1] - S.sfirst[J], m = S.rows_ptr[J + 1] - S.rows_ptr[J];
      const int32_t* r = S.rows.data() + S.rows_ptr[J];
      int32_t last = -1;
      for (int64_t qq = k; qq < m; ++qq) {
        int32_t P = S.snode[r[qq]];
        if (P != last) { pj.push_back(J); pp.push_back(P); pq.push_back((int32_t)qq); last = P; }
      }
      S.rel_ptr[J + 1] = (int64_t)pj.size();
    }
    const int64_t np = (int64_t)pj.size();
    S.rel_anc = pp; S.rel_q0 = pq;
    S.rel_off.assign(np + 1, 0);
    for (int64_t x = 0; x < np; ++x) S.rel_off[x + 1] = S.rel_off[x] + (S.rows_ptr[pj[x] + 1] - S.rows_ptr[pj[x]] - pq[x]);
    S.relind.assign(S.rel_off[np], 0);
    std::vector<int64_t> bp(ns + 1, 0);
    for (int64_t x = 0; x < np; ++x) bp[pp[x] + 1]++;
    for (int32_t s = 0; s < ns; ++s) bp[s + 1] += bp[s];
    std::vector<int64_t> byP(np);
    { std::vector<int64_t> nx(bp.begin(), bp.end() - 1); for (int64_t x = 0; x < np; ++x) byP[nx[pp[x]]++] = x; }
    std::vector<int32_t> indmap(n, 0);
    for (int32_t P = 0; P < ns; ++P) {
      if (bp[P] == bp[P + 1]) continue;
      int64_t mP = S.rows_ptr[P + 1] - S.rows_ptr[P];
      const int32_t* rP = S.rows.data() + S.rows_ptr[P];
      for (int64_t x = 0; x < mP; ++x) indmap[rP[x]] = (int32_t)(mP - 1 - x);   // distance from the bottom
      for (int64_t b = bp[P]; b < bp[P + 1]; ++b) {
        int64_t x = byP[b];
        int32_t J = pj[x];
        const int32_t* rJ = S.rows.data() + S.rows_ptr[J];
        int64_t m = S.rows_ptr[J + 1] - S.rows_ptr[J];
        int32_t* out = S.relind.data() + S.rel_off[x];
        for (int64_t qq = pq[x]; qq < m; ++qq) *out++ = indmap[rJ[qq]];
      }
    }
  }
  // ---- RLB blocks from the relind pairs: inside a pair's tail, a block breaks where the global
  // row is not the previous one + 1 (rows(P) positions then jump) or where the next pair starts
  {
    S.blk_ptr.assign(ns + 1, 0);
    S.blk_q.clear(); S.blk_len.clear(); S.blk_anc.clear(); S.blk_relind.clear();
    for (int32_t J = 0; J < ns; ++J) {
      const int32_t* rJ = S.rows.data() + S.rows_ptr[J];
      const int64_t m = S.rows_ptr[J + 1] - S.rows_ptr[J];
      for (int64_t x = S.rel_ptr[J]; x < S.rel_ptr[J + 1]; ++x) {
        const int64_t qend = x + 1 < S.rel_ptr[J + 1] ? S.rel_q0[x + 1] : m;   // rows of this ancestor
        for (int64_t qq = S.rel_q0[x]; qq < qend; ++qq) {
          const int32_t rel = S.relind[S.rel_off[x] + (qq - S.rel_q0[x])];
          if (qq == S.rel_q0[x] || rJ[qq] != rJ[qq - 1] + 1) {
            S.blk_q.push_back((int32_t)qq);
            S.blk_len.push_back(0);
            S.blk_anc.push_back(S.rel_anc[x]);
            S.blk_relind.push_back(rel);
          }
          S.blk_len.back()++;
        }
      }
      S.blk_ptr[J + 1] = (int64_t)S.blk_q.size();
    }
  }
  // ---- A entry -> (final column, position in rows(J))
  S.a_col.assign(S.nnzA, 0); S.a_pos.assign(S.nnzA, 0);
  {
    std::vector<int32_t> pos(n, 0);
    for (int32_t s = 0; s < ns; ++s) {
      int64_t m = S.rows_ptr[s + 1] - S.rows_ptr[s];
      const int32_t* r = S.rows.data() + S.rows_ptr[s];
      for (int64_t x = 0; x < m; ++x) pos[r[x]] = (int32_t)x;
      for (int32_t c = S.sfirst[s]; c < S.sfirst[s + 1]; ++c)
        for (int64_t p = Cf.cp[c]; p < Cf.cp[c + 1]; ++p) {
          int64_t e = Cf.src[p];
          S.a_col[e] = c;
          S.a_pos[e] = pos[Cf.ci[p]];
        }
    }
  }
  return SPCHOL_OK;
}

}  // namespace spchol
