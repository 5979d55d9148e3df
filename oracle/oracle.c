/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of what the product path computes
 * (SURVEY.md §8(c) steps O1-O10).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code with
 * paper_2409_14009_b200/ (no headers, helpers or tables); the only common module is gen/
 * (input generators).
 *
 * Compiled with -O2 -ffp-contract=off (no FMA contraction), IEEE FP64, round-to-nearest.
 *
 * Steps and the passages they follow (P:n = /root/reference/PAPER.md line n):
 *   O1 permute            C = P A P^T                                  (perm is an input)
 *   O2 symbolic           row-merge: struct(L_j) = {j} u {i>j: C_ij!=0} u U_{c: parent(c)=j} struct(L_c)\{c}
 *                         parent(j) = min(struct(L_j)\{j})
 *   O3 postorder          DFS from roots ascending, children ascending, number on exit
 *   O4 column counts      cc_j = |struct(L_j)|, nnz(L) = sum cc_j, F = sum cc_j^2
 *   O5 supernodes         fundamental [LNP93] (reading R1): j+1 joins j iff
 *                         parent(j)=j+1, cc_j = cc_{j+1}+1 and j+1 has exactly one child.
 *                         rule=1 gives the "maximal" partition of Fig. 1 (no child condition).
 *   O6 greedy merge       pairs (J, p(J)), minimum new fill first, stop before cumulative growth
 *                         exceeds cap * nnz(L)  (readings R3-R6)
 *   O7 final permutation  postorder of the merged supernodal tree (reading R6)
 *   O7b partition refinement (optional, pr = 1, reading R14): the
 *                         columns inside each supernode P are reordered: the ordered partition
 *                         [cols(P)] is refined by S_J = R_J n cols(P) for every J with S_J nonempty,
 *                         J ascending, each part X becoming (X n S_J, X \ S_J), order kept inside
 *   O8 relind             relind(J,P)[q] = (m_P - 1) - position of rows(J)[q] in rows(P),
 *                         for the rows of J that are >= f_P ("distance from the bottom")
 *   O9 numeric            scalar left-looking column Cholesky of C_f = P_f A P_f^T on its exact
 *                         structure (A = L L^T); the unique Cholesky factor.
 *   O8b RLB blocks        for each J, the rows below cols(J) split into maximal runs of consecutive
 *                         global rows lying in one ancestor's column range; per block:
 *                         first row position q in rows(J), length, ancestor P, relindB =
 *                         m_P - 1 - position of the block's first row in rows(P)
 *   O10 solve             L y = P_f b, L^T z = y, x = P_f^T z  ("triangular factors are used
 *                         to compute the solution")
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int64_t n;
  /* O3 / fundamental / merge (all in O3 numbering) */
  int32_t* post;      /* post[new3] = old (user-permuted numbering) */
  int32_t* parent3;   /* exact etree in O3 numbering */
  int32_t* cc3;       /* column counts in O3 numbering */
  int64_t nnzL;
  double flops;       /* sum cc^2 */
  int32_t nfund;
  int32_t* ffirst;    /* [nfund+1] fundamental partition, O3 numbering */
  int32_t* fparent;   /* fundamental supernodal parent (-1 = root) */
  int32_t* fgroup;    /* fundamental supernode -> merged group id (fundamental index of its top) */
  int64_t added;      /* storage added by merging */
  int32_t nmerges;
  int32_t* merge_child; int32_t* merge_parent; int64_t* merge_cost;  /* merge log */
  /* final (O7) numbering */
  int32_t* perm_final; /* perm_final[orig] = final */
  int32_t* o7;         /* o7[o3] = final */
  int32_t nsuper;
  int32_t* sfirst;     /* [nsuper+1] */
  int32_t* sparent;    /* merged supernodal parent, -1 = root */
  int64_t* rows_ptr;   /* [nsuper+1] */
  int32_t* rows;       /* rows(J), final numbering, ascending */
  int64_t* rel_ptr;    /* [nsuper+1] index into rel_list */
  int32_t* rel_anc;    /* per (J,P) pair: P */
  int32_t* rel_q0;     /* per pair: first q in rows(J) with rows(J)[q] >= f_P */
  int64_t* rel_off;    /* per pair: offset into relind */
  int64_t npairs;
  int32_t* relind;
  int64_t nblocks;
  int64_t* blk_ptr;    /* [nsuper+1] blocks of J */
  int32_t* blk_q;      /* first row position in rows(J) */
  int32_t* blk_len;
  int32_t* blk_anc;
  int32_t* blk_relind; /* relindB: m_P - 1 - position of the first row in rows(P) */
  int32_t* parent_final; /* exact etree in final numbering */
  int32_t* cc_final;
  /* exact structure of L in final numbering (only when requested) */
  int64_t* Lp; int32_t* Li; double* Lx;
  /* permuted input C_f (for numeric) */
  int64_t* Cp; int32_t* Ci; double* Cx;
  int numeric_done;
} orc_t;

/* ---------------- helpers ---------------- */
static int cmp_i32(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

/* O1: C = P A P^T in lower CSC (rows ascending).  perm[old] = new. */
static void permute_lower(int64_t n, const int64_t* Ap, const int32_t* Ai, const double* Ax,
                          const int32_t* perm, int64_t** Cp_out, int32_t** Ci_out, double** Cx_out) {
  int64_t nnz = Ap[n];
  int64_t* Cp = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  int32_t* Ci = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nnz ? nnz : 1));
  double* Cx = Ax ? (double*)malloc(sizeof(double) * (size_t)(nnz ? nnz : 1)) : NULL;
  for (int64_t j = 0; j < n; ++j)
    for (int64_t p = Ap[j]; p < Ap[j + 1]; ++p) {
      int32_t a = perm[Ai[p]], b = perm[j];
      int32_t col = a < b ? a : b;
      Cp[col + 1]++;
    }
  for (int64_t j = 0; j < n; ++j) Cp[j + 1] += Cp[j];
  int64_t* next = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
  memcpy(next, Cp, sizeof(int64_t) * (size_t)n);
  for (int64_t j = 0; j < n; ++j)
    for (int64_t p = Ap[j]; p < Ap[j + 1]; ++p) {
      int32_t a = perm[Ai[p]], b = perm[j];
      int32_t col = a < b ? a : b, row = a < b ? b : a;
      int64_t q = next[col]++;
      Ci[q] = row;
      if (Cx) Cx[q] = Ax[p];
    }
  free(next);
  /* sort rows within each column (insertion sort; columns are short) */
  for (int64_t j = 0; j < n; ++j) {
    for (int64_t p = Cp[j] + 1; p < Cp[j + 1]; ++p) {
      int32_t r = Ci[p]; double v = Cx ? Cx[p] : 0.0; int64_t q = p - 1;
      while (q >= Cp[j] && Ci[q] > r) { Ci[q + 1] = Ci[q]; if (Cx) Cx[q + 1] = Cx[q]; --q; }
      Ci[q + 1] = r; if (Cx) Cx[q + 1] = v;
    }
  }
  *Cp_out = Cp; *Ci_out = Ci; if (Cx_out) *Cx_out = Cx; else free(Cx);
}

/*
 * O2: symbolic factorization by row-merge.  Computes parent and cc for every column.
 * keep[j] != 0 (or keep == NULL && keep_all) retains struct(L_j) sorted in (*Sp, *Si).
 * Structures of columns that are not kept are freed as soon as their parent consumed them.
 */
static int rowmerge(int64_t n, const int64_t* Cp, const int32_t* Ci, int32_t* parent, int32_t* cc,
                    const char* keep, int keep_all, int64_t** Sp_out, int32_t** Si_out) {
  int32_t** st = (int32_t**)calloc((size_t)n + 1, sizeof(int32_t*));
  int32_t* len = (int32_t*)calloc((size_t)n + 1, sizeof(int32_t));
  int32_t* mark = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1));
  int32_t* buf = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1));
  /* children lists: head/next over columns */
  int32_t* chead = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1));
  int32_t* cnext = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1));
  int32_t* ctail = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1));
  if (!st || !len || !mark || !buf || !chead || !cnext || !ctail) return -1;
  for (int64_t j = 0; j < n; ++j) { mark[j] = -1; chead[j] = -1; ctail[j] = -1; cnext[j] = -1; }
  for (int64_t j = 0; j < n; ++j) {
    int32_t cnt = 0;
    buf[cnt++] = (int32_t)j; mark[j] = (int32_t)j;
    for (int64_t p = Cp[j]; p < Cp[j + 1]; ++p) {
      int32_t i = Ci[p];
      if (i > j && mark[i] != j) { mark[i] = (int32_t)j; buf[cnt++] = i; }
    }
    for (int32_t c = chead[j]; c != -1; c = cnext[c]) {
      for (int32_t q = 0; q < len[c]; ++q) {
        int32_t i = st[c][q];
        if (i != c && mark[i] != j) { mark[i] = (int32_t)j; buf[cnt++] = i; }
      }
      if (!(keep_all || (keep && keep[c]))) { free(st[c]); st[c] = NULL; }
    }
    int32_t par = -1;
    for (int32_t q = 1; q < cnt; ++q) if (par == -1 || buf[q] < par) par = buf[q];
    parent[j] = par; cc[j] = cnt;
    st[j] = (int32_t*)malloc(sizeof(int32_t) * (size_t)cnt);
    memcpy(st[j], buf, sizeof(int32_t) * (size_t)cnt);
    qsort(st[j], (size_t)cnt, sizeof(int32_t), cmp_i32);
    len[j] = cnt;
    if (par != -1) {  /* append j to parent's child list (ascending) */
      if (ctail[par] == -1) chead[par] = (int32_t)j; else cnext[ctail[par]] = (int32_t)j;
      ctail[par] = (int32_t)j;
    }
  }
  int64_t* Sp = NULL; int32_t* Si = NULL;
  if (Sp_out) {
    Sp = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
    for (int64_t j = 0; j < n; ++j) Sp[j + 1] = Sp[j] + ((keep_all || (keep && keep[j])) ? len[j] : 0);
    Si = (int32_t*)malloc(sizeof(int32_t) * (size_t)(Sp[n] ? Sp[n] : 1));
    for (int64_t j = 0; j < n; ++j)
      if (keep_all || (keep && keep[j])) memcpy(Si + Sp[j], st[j], sizeof(int32_t) * (size_t)len[j]);
    *Sp_out = Sp; *Si_out = Si;
  }
  for (int64_t j = 0; j < n; ++j) free(st[j]);
  free(st); free(len); free(mark); free(buf); free(chead); free(cnext); free(ctail);
  return 0;
}

/* O3: postorder; post[k] = node numbered k. */
static void postorder(int64_t n, const int32_t* parent, int32_t* post) {
  int32_t* head = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1));
  int32_t* next = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1));
  int32_t* stack = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1));
  for (int64_t j = 0; j < n; ++j) head[j] = -1;
  /* children ascending: insert in descending order at the head */
  for (int64_t j = n - 1; j >= 0; --j)
    if (parent[j] != -1) { next[j] = head[parent[j]]; head[parent[j]] = (int32_t)j; }
  int64_t k = 0;
  for (int64_t r = 0; r < n; ++r) {
    if (parent[r] != -1) continue;
    int64_t top = 0; stack[top++] = (int32_t)r;
    while (top > 0) {
      int32_t v = stack[top - 1];
      int32_t c = head[v];
      if (c == -1) { post[k++] = v; --top; }
      else { head[v] = next[c]; stack[top++] = c; }
    }
  }
  free(head); free(next); free(stack);
}

/* ---------------- lazy min-heap of (cost, id) for O6 ---------------- */
typedef struct { int64_t cost; int32_t id; } hent;
typedef struct { hent* a; int64_t n, cap; } heap_t;
static int hless(hent x, hent y) { return x.cost < y.cost || (x.cost == y.cost && x.id < y.id); }
static void hpush(heap_t* h, hent e) {
  if (h->n == h->cap) { h->cap = h->cap ? 2 * h->cap : 1024; h->a = (hent*)realloc(h->a, sizeof(hent) * (size_t)h->cap); }
  int64_t i = h->n++;
  h->a[i] = e;
  while (i > 0) { int64_t p = (i - 1) / 2; if (!hless(h->a[i], h->a[p])) break; hent t = h->a[i]; h->a[i] = h->a[p]; h->a[p] = t; i = p; }
}
static hent hpop(heap_t* h) {
  hent top = h->a[0];
  h->a[0] = h->a[--h->n];
  int64_t i = 0;
  for (;;) {
    int64_t l = 2 * i + 1, r = l + 1, m = i;
    if (l < h->n && hless(h->a[l], h->a[m])) m = l;
    if (r < h->n && hless(h->a[r], h->a[m])) m = r;
    if (m == i) break;
    hent t = h->a[i]; h->a[i] = h->a[m]; h->a[m] = t; i = m;
  }
  return top;
}
static int32_t uf_find(int32_t* uf, int32_t x) {
  int32_t r = x;
  while (uf[r] != r) r = uf[r];
  while (uf[x] != r) { int32_t nx = uf[x]; uf[x] = r; x = nx; }
  return r;
}

/* ---------------- public API ---------------- */
void orc_free(orc_t* o);

/*
 * Symbolic phase O1-O8.  rule: 0 fundamental, 1 maximal.  cap < 0 disables merging.
 * keep_L: also build the exact structure of L in final numbering (needed by orc_numeric).
 * values may be NULL (then orc_numeric is unavailable).
 */
orc_t* orc_symbolic_pr(int64_t n, const int64_t* Ap, const int32_t* Ai, const double* Ax,
                       const int32_t* perm, double cap, int rule, int keep_L, int pr);
orc_t* orc_symbolic(int64_t n, const int64_t* Ap, const int32_t* Ai, const double* Ax,
                    const int32_t* perm, double cap, int rule, int keep_L) {
  return orc_symbolic_pr(n, Ap, Ai, Ax, perm, cap, rule, keep_L, 0);
}

/*
 * O7b (reading R14): partition refinement of the columns inside every supernode.  Input: the O7
 * supernodes (sfirst) and rows(J) in O7 labels.  Output newlab[O7 label] = refined label.  Plain
 * version: the whole ordered partition of P is rebuilt for every refining set.
 */
static void partition_refinement(int64_t n, int32_t ns, const int32_t* sfirst, const int64_t* rows_ptr,
                                 const int32_t* rows, int32_t* newlab) {
  int32_t* snode = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
  for (int32_t s = 0; s < ns; ++s) for (int32_t c = sfirst[s]; c < sfirst[s + 1]; ++c) snode[c] = s;
  int32_t* ord = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));     /* per P: its columns in order */
  char* brk = (char*)calloc((size_t)n + 1, 1);                                  /* brk[i]: a part starts at ord[i] */
  char* inS = (char*)calloc((size_t)n + 1, 1);
  int32_t* tmp = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
  char* tbrk = (char*)calloc((size_t)n + 1, 1);
  for (int64_t c = 0; c < n; ++c) ord[c] = (int32_t)c;
  for (int32_t s = 0; s < ns; ++s) brk[sfirst[s]] = 1;
  for (int32_t J = 0; J < ns; ++J) {
    int64_t k = sfirst[J + 1] - sfirst[J];
    for (int64_t q = rows_ptr[J] + k; q < rows_ptr[J + 1];) {
      int32_t P = snode[rows[q]];
      int64_t q1 = q;
      while (q1 < rows_ptr[J + 1] && snode[rows[q1]] == P) { inS[rows[q1]] = 1; ++q1; }   /* S_J */
      /* rebuild P's ordered partition: every part X -> (X n S_J, X \ S_J) */
      int32_t a = sfirst[P], b = sfirst[P + 1], w = a;
      for (int32_t i = a; i < b;) {
        int32_t e = i + 1;
        while (e < b && !brk[e]) ++e;                 /* part [i, e) */
        int32_t w0 = w;
        for (int32_t x = i; x < e; ++x) if (inS[ord[x]]) tmp[w++] = ord[x];
        int32_t w1 = w;
        for (int32_t x = i; x < e; ++x) if (!inS[ord[x]]) tmp[w++] = ord[x];
        if (w1 > w0) tbrk[w0] = 1;
        if (w > w1) tbrk[w1] = 1;
        i = e;
      }
      for (int32_t i = a; i < b; ++i) { ord[i] = tmp[i]; brk[i] = tbrk[i]; tbrk[i] = 0; }
      for (int64_t x = q; x < q1; ++x) inS[rows[x]] = 0;
      q = q1;
    }
  }
  for (int64_t i = 0; i < n; ++i) newlab[ord[i]] = (int32_t)i;
  free(snode); free(ord); free(brk); free(inS); free(tmp); free(tbrk);
}

orc_t* orc_symbolic_pr(int64_t n, const int64_t* Ap, const int32_t* Ai, const double* Ax,
                       const int32_t* perm, double cap, int rule, int keep_L, int pr) {
  orc_t* o = (orc_t*)calloc(1, sizeof(orc_t));
  o->n = n;
  int32_t* ident = NULL;
  if (!perm) { ident = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1)); for (int64_t i = 0; i < n; ++i) ident[i] = (int32_t)i; perm = ident; }
  /* O1 */
  int64_t *Cp; int32_t* Ci;
  permute_lower(n, Ap, Ai, NULL, perm, &Cp, &Ci, NULL);
  /* O2 on C */
  int32_t* parent = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
  int32_t* cc = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
  rowmerge(n, Cp, Ci, parent, cc, NULL, 0, NULL, NULL);
  /* O3 */
  o->post = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
  postorder(n, parent, o->post);
  int32_t* ipost = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
  for (int64_t k = 0; k < n; ++k) ipost[o->post[k]] = (int32_t)k;
  o->parent3 = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
  o->cc3 = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
  for (int64_t j = 0; j < n; ++j) {
    o->parent3[ipost[j]] = parent[j] == -1 ? -1 : ipost[parent[j]];
    o->cc3[ipost[j]] = cc[j];
  }
  /* O4 */
  o->nnzL = 0; o->flops = 0.0;
  for (int64_t j = 0; j < n; ++j) { o->nnzL += o->cc3[j]; o->flops += (double)o->cc3[j] * (double)o->cc3[j]; }
  /* O5 in O3 numbering */
  int32_t* nchild = (int32_t*)calloc((size_t)n + 1, sizeof(int32_t));
  for (int64_t j = 0; j < n; ++j) if (o->parent3[j] != -1) nchild[o->parent3[j]]++;
  o->ffirst = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1));
  int32_t* fsn = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));  /* column -> fundamental */
  int32_t nf = 0;
  for (int64_t j = 0; j < n; ++j) {
    int join = j > 0 && o->parent3[j - 1] == j && o->cc3[j - 1] == o->cc3[j] + 1 && (rule == 1 || nchild[j] == 1);
    if (!join) o->ffirst[nf++] = (int32_t)j;
    fsn[j] = nf - 1;
  }
  o->ffirst[nf] = (int32_t)n;
  o->nfund = nf;
  o->fparent = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nf ? nf : 1));
  for (int32_t f = 0; f < nf; ++f) {
    int32_t last = o->ffirst[f + 1] - 1;
    o->fparent[f] = o->parent3[last] == -1 ? -1 : fsn[o->parent3[last]];
  }
  /* rows of the fundamental heads: second row-merge on C3 = Q C Q^T keeping only head columns */
  int64_t *C3p; int32_t* C3i;
  {
    int32_t* q = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
    for (int64_t i = 0; i < n; ++i) q[i] = ipost[i];
    permute_lower(n, Cp, Ci, NULL, q, &C3p, &C3i, NULL);
    free(q);
  }
  char* keep = (char*)calloc((size_t)n + 1, 1);
  for (int32_t f = 0; f < nf; ++f) keep[o->ffirst[f]] = 1;
  int32_t* par2 = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
  int32_t* cc2 = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
  int64_t* Hp; int32_t* Hi;
  rowmerge(n, C3p, C3i, par2, cc2, keep, 0, &Hp, &Hi);
  for (int64_t j = 0; j < n; ++j)
    if (par2[j] != o->parent3[j] || cc2[j] != o->cc3[j]) { /* self-check: relabelling must commute */
      orc_free(o); o = NULL; goto done_early;
    }
  /* O6 greedy merge over the fundamental supernodal tree */
  {
    int64_t* k = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nf ? nf : 1));
    int64_t* m = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nf ? nf : 1));
    int32_t* uf = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nf ? nf : 1));
    char* alive = (char*)malloc((size_t)(nf ? nf : 1));
    for (int32_t f = 0; f < nf; ++f) {
      k[f] = o->ffirst[f + 1] - o->ffirst[f];
      m[f] = o->cc3[o->ffirst[f]];
      uf[f] = f; alive[f] = 1;
    }
    o->merge_child = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nf ? nf : 1));
    o->merge_parent = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nf ? nf : 1));
    o->merge_cost = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nf ? nf : 1));
    heap_t h = {0};
    double budget = cap * (double)o->nnzL;
    if (cap >= 0) {
      for (int32_t f = 0; f < nf; ++f)
        if (o->fparent[f] != -1) {
          int32_t P = o->fparent[f];
          hent e = {k[f] * (k[f] + m[P] - m[f]), f};
          hpush(&h, e);
        }
    }
    int64_t added = 0;
    while (h.n > 0) {
      hent e = hpop(&h);
      int32_t J = e.id;
      if (!alive[J]) continue;
      int32_t P = uf_find(uf, o->fparent[J]);
      int64_t cost = k[J] * (k[J] + m[P] - m[J]);
      if (cost != e.cost) { hent e2 = {cost, J}; hpush(&h, e2); continue; }
      if ((double)(added + cost) > budget) break;   /* never exceed the cap */
      o->merge_child[o->nmerges] = J; o->merge_parent[o->nmerges] = P; o->merge_cost[o->nmerges] = cost; o->nmerges++;
      added += cost;
      m[P] = k[J] + m[P];
      k[P] = k[J] + k[P];
      alive[J] = 0; uf[J] = P;
    }
    free(h.a);
    o->added = added;
    o->fgroup = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nf ? nf : 1));
    for (int32_t f = 0; f < nf; ++f) o->fgroup[f] = uf_find(uf, f);
    free(k); free(m); free(uf); free(alive);
  }
  /* O7 final permutation: postorder of the merged tree */
  {
    /* group ids are the fundamental indices of alive tops */
    int32_t* gparent = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nf ? nf : 1));
    int32_t* gmin = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nf ? nf : 1));
    for (int32_t f = 0; f < nf; ++f) { gparent[f] = -2; gmin[f] = INT32_MAX; }
    for (int32_t f = 0; f < nf; ++f) {
      int32_t g = o->fgroup[f];
      if (o->ffirst[f] < gmin[g]) gmin[g] = o->ffirst[f];
      if (g == f) gparent[g] = o->fparent[f] == -1 ? -1 : o->fgroup[o->fparent[f]];
    }
    /* groups sorted by smallest O3 column: order children/roots by gmin */
    int32_t ng = 0;
    int32_t* gl = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nf ? nf : 1));
    for (int32_t f = 0; f < nf; ++f) if (o->fgroup[f] == f) gl[ng++] = f;
    /* sort gl by gmin (simple: gmin values are distinct column indices) */
    int32_t* bycol = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
    for (int64_t j = 0; j < n; ++j) bycol[j] = -1;
    for (int32_t a = 0; a < ng; ++a) bycol[gmin[gl[a]]] = gl[a];
    ng = 0;
    for (int64_t j = 0; j < n; ++j) if (bycol[j] != -1) gl[ng++] = bycol[j];
    free(bycol);
    /* children lists in gmin-ascending order */
    int32_t* head = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nf ? nf : 1));
    int32_t* nxt = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nf ? nf : 1));
    for (int32_t f = 0; f < nf; ++f) head[f] = -1;
    for (int32_t a = ng - 1; a >= 0; --a) {
      int32_t g = gl[a];
      if (gparent[g] >= 0) { nxt[g] = head[gparent[g]]; head[gparent[g]] = g; }
    }
    /* member columns of each group, ascending */
    int64_t* gcnt = (int64_t*)calloc((size_t)nf + 1, sizeof(int64_t));
    for (int64_t j = 0; j < n; ++j) gcnt[o->fgroup[fsn[j]] + 1]++;
    for (int32_t f = 0; f < nf; ++f) gcnt[f + 1] += gcnt[f];
    int32_t* gcols = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
    int64_t* gpos = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nf + 1));
    memcpy(gpos, gcnt, sizeof(int64_t) * (size_t)(nf + 1));
    for (int64_t j = 0; j < n; ++j) gcols[gpos[o->fgroup[fsn[j]]]++] = (int32_t)j;  /* ascending j */
    free(gpos);
    o->o7 = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
    o->sfirst = (int32_t*)malloc(sizeof(int32_t) * (size_t)(ng + 1));
    int32_t* gsuper = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nf ? nf : 1));
    int32_t* stack = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nf ? nf : 1));
    int32_t* hd = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nf ? nf : 1));
    memcpy(hd, head, sizeof(int32_t) * (size_t)(nf ? nf : 1));
    int32_t counter = 0, ns = 0;
    for (int32_t a = 0; a < ng; ++a) {
      int32_t r = gl[a];
      if (gparent[r] != -1) continue;
      int32_t top = 0; stack[top++] = r;
      while (top > 0) {
        int32_t v = stack[top - 1];
        int32_t c = hd[v];
        if (c == -1) {
          --top;
          gsuper[v] = ns; o->sfirst[ns++] = counter;
          for (int64_t p = gcnt[v]; p < gcnt[v + 1]; ++p) o->o7[gcols[p]] = counter++;
        } else { hd[v] = nxt[c]; stack[top++] = c; }
      }
    }
    o->sfirst[ns] = counter;
    o->nsuper = ns;
    o->sparent = (int32_t*)malloc(sizeof(int32_t) * (size_t)(ns ? ns : 1));
    for (int32_t a = 0; a < ng; ++a) {
      int32_t g = gl[a];
      o->sparent[gsuper[g]] = gparent[g] == -1 ? -1 : gsuper[gparent[g]];
    }
    /* rows(J) = cols(J) u rows(top fundamental member) in final numbering */
    o->rows_ptr = (int64_t*)calloc((size_t)ns + 1, sizeof(int64_t));
    int32_t* gof = (int32_t*)malloc(sizeof(int32_t) * (size_t)(ns ? ns : 1)); /* super -> group id */
    for (int32_t a = 0; a < ng; ++a) gof[gsuper[gl[a]]] = gl[a];
    for (int32_t s = 0; s < ns; ++s) {
      int32_t g = gof[s];
      int64_t kg = gcnt[g + 1] - gcnt[g];
      int64_t mtop = Hp[o->ffirst[g] + 1] - Hp[o->ffirst[g]];
      int64_t ktop = o->ffirst[g + 1] - o->ffirst[g];
      o->rows_ptr[s + 1] = o->rows_ptr[s] + (kg - ktop) + mtop;
    }
    o->rows = (int32_t*)malloc(sizeof(int32_t) * (size_t)(o->rows_ptr[ns] ? o->rows_ptr[ns] : 1));
    for (int32_t s = 0; s < ns; ++s) {
      int32_t g = gof[s];
      int64_t w = o->rows_ptr[s];
      for (int64_t p = gcnt[g]; p < gcnt[g + 1]; ++p) {
        int32_t c = gcols[p];
        if (fsn[c] != g) o->rows[w++] = o->o7[c];
      }
      for (int64_t p = Hp[o->ffirst[g]]; p < Hp[o->ffirst[g] + 1]; ++p) o->rows[w++] = o->o7[Hi[p]];
      qsort(o->rows + o->rows_ptr[s], (size_t)(w - o->rows_ptr[s]), sizeof(int32_t), cmp_i32);
    }
    free(gof); free(stack); free(hd); free(head); free(nxt); free(gcnt); free(gcols); free(gsuper);
    free(gparent); free(gmin); free(gl);
  }
  /* O7b partition refinement: relabel the columns inside each supernode, rows(J) re-sorted */
  if (pr) {
    int32_t* newlab = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
    partition_refinement(n, o->nsuper, o->sfirst, o->rows_ptr, o->rows, newlab);
    for (int64_t j = 0; j < n; ++j) o->o7[j] = newlab[o->o7[j]];
    for (int64_t x = 0; x < o->rows_ptr[o->nsuper]; ++x) o->rows[x] = newlab[o->rows[x]];
    for (int32_t s = 0; s < o->nsuper; ++s)
      qsort(o->rows + o->rows_ptr[s], (size_t)(o->rows_ptr[s + 1] - o->rows_ptr[s]), sizeof(int32_t), cmp_i32);
    free(newlab);
  }
  /* final permutation and exact etree / cc in final numbering */
  o->perm_final = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
  for (int64_t i = 0; i < n; ++i) o->perm_final[i] = o->o7[ipost[perm[i]]];
  o->parent_final = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
  o->cc_final = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
  if (!pr) {   /* O7 is an equivalent (topological) reordering: the O3 etree relabelled */
    for (int64_t j = 0; j < n; ++j) {
      o->parent_final[o->o7[j]] = o->parent3[j] == -1 ? -1 : o->o7[o->parent3[j]];
      o->cc_final[o->o7[j]] = o->cc3[j];
    }
  } else {     /* a reordering inside supernodes can change the exact structure: row-merge again */
    int64_t *Fp; int32_t* Fi;
    permute_lower(n, Ap, Ai, NULL, o->perm_final, &Fp, &Fi, NULL);
    rowmerge(n, Fp, Fi, o->parent_final, o->cc_final, NULL, 0, NULL, NULL);
    free(Fp); free(Fi);
    o->nnzL = 0; o->flops = 0.0;   /* the exact factor actually computed */
    for (int64_t j = 0; j < n; ++j) { o->nnzL += o->cc_final[j]; o->flops += (double)o->cc_final[j] * (double)o->cc_final[j]; }
  }
  /* O8 relind */
  {
    int32_t ns = o->nsuper;
    int32_t* snode = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
    for (int32_t s = 0; s < ns; ++s) for (int32_t c = o->sfirst[s]; c < o->sfirst[s + 1]; ++c) snode[c] = s;
    o->rel_ptr = (int64_t*)calloc((size_t)ns + 1, sizeof(int64_t));
    /* count pairs and relind length */
    int64_t np = 0, nr = 0;
    for (int32_t J = 0; J < ns; ++J) {
      int64_t k = o->sfirst[J + 1] - o->sfirst[J];
      int64_t m = o->rows_ptr[J + 1] - o->rows_ptr[J];
      int32_t last = -1;
      for (int64_t q = k; q < m; ++q) {
        int32_t P = snode[o->rows[o->rows_ptr[J] + q]];
        if (P != last) { np++; nr += m - q; last = P; }
      }
      o->rel_ptr[J + 1] = np;
    }
    o->npairs = np;
    o->rel_anc = (int32_t*)malloc(sizeof(int32_t) * (size_t)(np ? np : 1));
    o->rel_q0 = (int32_t*)malloc(sizeof(int32_t) * (size_t)(np ? np : 1));
    o->rel_off = (int64_t*)malloc(sizeof(int64_t) * (size_t)(np + 1));
    o->relind = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nr ? nr : 1));
    int32_t* indmap = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
    int64_t pi = 0, ri = 0;
    for (int32_t J = 0; J < ns; ++J) {
      int64_t k = o->sfirst[J + 1] - o->sfirst[J];
      int64_t m = o->rows_ptr[J + 1] - o->rows_ptr[J];
      const int32_t* rJ = o->rows + o->rows_ptr[J];
      int32_t last = -1;
      for (int64_t q = k; q < m; ++q) {
        int32_t P = snode[rJ[q]];
        if (P == last) continue;
        last = P;
        int64_t mP = o->rows_ptr[P + 1] - o->rows_ptr[P];
        const int32_t* rP = o->rows + o->rows_ptr[P];
        for (int64_t x = 0; x < mP; ++x) indmap[rP[x]] = (int32_t)(mP - 1 - x);   /* indmap */
        o->rel_anc[pi] = P; o->rel_q0[pi] = (int32_t)q; o->rel_off[pi] = ri;
        for (int64_t qq = q; qq < m; ++qq) o->relind[ri++] = indmap[rJ[qq]];
        ++pi;
      }
    }
    o->rel_off[np] = ri;
    free(indmap); free(snode);
  }
  /* O8b RLB blocks: maximal runs of consecutive global rows of R_J inside one ancestor */
  {
    int32_t ns = o->nsuper;
    int32_t* snode = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
    for (int32_t s2 = 0; s2 < ns; ++s2) for (int32_t c = o->sfirst[s2]; c < o->sfirst[s2 + 1]; ++c) snode[c] = s2;
    o->blk_ptr = (int64_t*)calloc((size_t)ns + 1, sizeof(int64_t));
    int64_t nb = 0;
    for (int32_t J = 0; J < ns; ++J) {
      int64_t k = o->sfirst[J + 1] - o->sfirst[J], m = o->rows_ptr[J + 1] - o->rows_ptr[J];
      const int32_t* r = o->rows + o->rows_ptr[J];
      for (int64_t q = k; q < m; ++q)
        if (q == k || r[q] != r[q - 1] + 1 || snode[r[q]] != snode[r[q - 1]]) nb++;
      o->blk_ptr[J + 1] = nb;
    }
    o->nblocks = nb;
    o->blk_q = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nb ? nb : 1));
    o->blk_len = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nb ? nb : 1));
    o->blk_anc = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nb ? nb : 1));
    o->blk_relind = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nb ? nb : 1));
    int64_t b = 0;
    for (int32_t J = 0; J < ns; ++J) {
      int64_t k = o->sfirst[J + 1] - o->sfirst[J], m = o->rows_ptr[J + 1] - o->rows_ptr[J];
      const int32_t* r = o->rows + o->rows_ptr[J];
      for (int64_t q = k; q < m; ++q) {
        if (q == k || r[q] != r[q - 1] + 1 || snode[r[q]] != snode[r[q - 1]]) {
          int32_t P = snode[r[q]];
          int64_t mP = o->rows_ptr[P + 1] - o->rows_ptr[P];
          const int32_t* rP = o->rows + o->rows_ptr[P];
          int64_t pos = 0;
          while (rP[pos] != r[q]) ++pos;                 /* linear search: plain and obvious */
          o->blk_q[b] = (int32_t)q; o->blk_len[b] = 0; o->blk_anc[b] = P; o->blk_relind[b] = (int32_t)(mP - 1 - pos);
          ++b;
        }
        o->blk_len[b - 1]++;
      }
    }
    free(snode);
  }
  if (keep_L) {
    /* exact structure of L for C_f = P_f A P_f^T, plus the permuted values */
    permute_lower(n, Ap, Ai, Ax, o->perm_final, &o->Cp, &o->Ci, Ax ? &o->Cx : NULL);
    int32_t* p4 = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
    int32_t* c4 = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
    rowmerge(n, o->Cp, o->Ci, p4, c4, NULL, 1, &o->Lp, &o->Li);
    for (int64_t j = 0; j < n; ++j)
      if (p4[j] != o->parent_final[j] || c4[j] != o->cc_final[j]) { free(p4); free(c4); orc_free(o); o = NULL; goto done_early; }
    free(p4); free(c4);
  }
done_early:
  free(nchild); free(fsn); free(keep); free(par2); free(cc2); free(Hp); free(Hi);
  free(C3p); free(C3i); free(Cp); free(Ci); free(parent); free(cc); free(ipost); free(ident);
  return o;
}

/*
 * O9: scalar left-looking column Cholesky on the exact structure (George-Liu row lists).
 * Returns 0, or -3 with *fail_col = first column whose pivot is not > 0.
 * ncols < n factors only the leading ncols columns' dependencies... (full factor when ncols = n).
 */
int orc_numeric(orc_t* o, int64_t* fail_col) {
  int64_t n = o->n;
  *fail_col = -1;
  if (!o->Lp || !o->Cx) return -2;
  if (!o->Lx) o->Lx = (double*)malloc(sizeof(double) * (size_t)(o->Lp[n] ? o->Lp[n] : 1));
  double* w = (double*)calloc((size_t)n + 1, sizeof(double));
  int32_t* head = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1));
  int32_t* next = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1));
  int64_t* pos = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  int32_t* list = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1));
  for (int64_t j = 0; j < n; ++j) head[j] = -1;
  const int64_t* Lp = o->Lp; const int32_t* Li = o->Li; double* Lx = o->Lx;
  int rc = 0;
  for (int64_t j = 0; j < n; ++j) {
    /* w = C_f(:, j) (lower part) */
    for (int64_t p = o->Cp[j]; p < o->Cp[j + 1]; ++p) w[o->Ci[p]] = o->Cx[p];
    /* the columns k < j with L(j,k) != 0, ascending */
    int32_t cnt = 0;
    for (int32_t k = head[j]; k != -1; k = next[k]) list[cnt++] = k;
    qsort(list, (size_t)cnt, sizeof(int32_t), cmp_i32);
    head[j] = -1;
    for (int32_t a = 0; a < cnt; ++a) {
      int32_t k = list[a];
      int64_t pk = pos[k];            /* Li[pk] == j */
      double ljk = Lx[pk];
      for (int64_t p = pk; p < Lp[k + 1]; ++p) w[Li[p]] -= Lx[p] * ljk;
      /* move k to the list of its next row */
      if (pk + 1 < Lp[k + 1]) { pos[k] = pk + 1; int32_t r = Li[pk + 1]; next[k] = head[r]; head[r] = k; }
    }
    double d = w[j];
    if (!(d > 0.0)) { *fail_col = j; rc = -3; break; }
    double ljj = sqrt(d);
    Lx[Lp[j]] = ljj;  /* Li[Lp[j]] == j */
    w[j] = 0.0;
    for (int64_t p = Lp[j] + 1; p < Lp[j + 1]; ++p) { Lx[p] = w[Li[p]] / ljj; w[Li[p]] = 0.0; }
    if (Lp[j] + 1 < Lp[j + 1]) { pos[j] = Lp[j] + 1; int32_t r = Li[Lp[j] + 1]; next[j] = head[r]; head[r] = (int32_t)j; }
  }
  free(w); free(head); free(next); free(pos); free(list);
  o->numeric_done = rc == 0;
  return rc;
}

/*
 * O9, level-parallel build (the separately timed CPU baseline, SURVEY §8(d) "oracle-timed"): the
 * same scalar column computation as orc_numeric — w = C_f(:,j); for every k < j with L(j,k) != 0,
 * ascending, w -= L(:,k) L(j,k); pivot; scale — so every column is computed with the same
 * operations in the same order and L is bit-identical to the serial build.  Columns of equal
 * height in the elimination tree depend only on lower heights, so each height level is
 * split over nthreads POSIX threads (dynamic column assignment, one private accumulator each).
 * Returns as orc_numeric; *fail_col = the smallest failing column (the serial first failure:
 * a column computed from a failed one is larger, it is an ancestor).
 */
#include <pthread.h>
typedef struct {
  orc_t* o;
  const int64_t* rp; const int32_t* rk; const int64_t* rpos;   /* row lists: (k, position of j in column k) */
  const int32_t* lvl_cols; int64_t lo, hi;                    /* current level's columns */
  int64_t next;                                               /* next column index (atomic) */
  int64_t fail;                                               /* smallest failing column so far */
  pthread_mutex_t mu;
  pthread_barrier_t bar_start, bar_end;
  int stop;
} par_t;
typedef struct { par_t* P; double* w; } par_arg_t;

static void par_column(par_t* P, double* w, int64_t j) {
  orc_t* o = P->o;
  const int64_t* Lp = o->Lp; const int32_t* Li = o->Li; double* Lx = o->Lx;
  for (int64_t p = o->Cp[j]; p < o->Cp[j + 1]; ++p) w[o->Ci[p]] = o->Cx[p];
  for (int64_t a = P->rp[j]; a < P->rp[j + 1]; ++a) {
    int32_t k = P->rk[a];
    int64_t pk = P->rpos[a];          /* Li[pk] == j */
    double ljk = Lx[pk];
    for (int64_t p = pk; p < Lp[k + 1]; ++p) w[Li[p]] -= Lx[p] * ljk;
  }
  double d = w[j];
  w[j] = 0.0;
  if (!(d > 0.0)) {
    pthread_mutex_lock(&P->mu);
    if (P->fail < 0 || j < P->fail) P->fail = j;
    pthread_mutex_unlock(&P->mu);
    for (int64_t p = Lp[j] + 1; p < Lp[j + 1]; ++p) w[Li[p]] = 0.0;
    Lx[Lp[j]] = NAN;
    for (int64_t p = Lp[j] + 1; p < Lp[j + 1]; ++p) Lx[p] = NAN;
    return;
  }
  double ljj = sqrt(d);
  Lx[Lp[j]] = ljj;
  for (int64_t p = Lp[j] + 1; p < Lp[j + 1]; ++p) { Lx[p] = w[Li[p]] / ljj; w[Li[p]] = 0.0; }
}

static void* par_worker(void* arg) {
  par_arg_t* A = (par_arg_t*)arg;
  par_t* P = A->P;
  for (;;) {
    pthread_barrier_wait(&P->bar_start);
    if (P->stop) break;
    for (;;) {
      int64_t i = __atomic_fetch_add(&P->next, 1, __ATOMIC_RELAXED);
      if (i >= P->hi) break;
      par_column(P, A->w, P->lvl_cols[i]);
    }
    pthread_barrier_wait(&P->bar_end);
  }
  return NULL;
}

int orc_numeric_parallel(orc_t* o, int nthreads, int64_t* fail_col) {
  int64_t n = o->n;
  *fail_col = -1;
  if (!o->Lp || !o->Cx) return -2;
  if (nthreads < 1) nthreads = 1;
  if (!o->Lx) o->Lx = (double*)malloc(sizeof(double) * (size_t)(o->Lp[n] ? o->Lp[n] : 1));
  const int64_t* Lp = o->Lp; const int32_t* Li = o->Li;
  /* row lists of L (k ascending, as the serial build takes them) */
  int64_t* rp = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  for (int64_t k = 0; k < n; ++k) for (int64_t p = Lp[k] + 1; p < Lp[k + 1]; ++p) rp[Li[p] + 1]++;
  for (int64_t j = 0; j < n; ++j) rp[j + 1] += rp[j];
  int32_t* rk = (int32_t*)malloc(sizeof(int32_t) * (size_t)(rp[n] ? rp[n] : 1));
  int64_t* rpos = (int64_t*)malloc(sizeof(int64_t) * (size_t)(rp[n] ? rp[n] : 1));
  int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
  for (int64_t j = 0; j < n; ++j) fill[j] = rp[j];
  for (int64_t k = 0; k < n; ++k)
    for (int64_t p = Lp[k] + 1; p < Lp[k + 1]; ++p) { int32_t i = Li[p]; rk[fill[i]] = (int32_t)k; rpos[fill[i]++] = p; }
  /* etree heights (parent > child), columns grouped by height */
  int32_t* h = (int32_t*)calloc((size_t)n + 1, sizeof(int32_t));
  int32_t H = 0;
  for (int64_t j = 0; j < n; ++j) {
    int32_t par = o->parent_final[j];
    if (par >= 0 && h[par] < h[j] + 1) h[par] = h[j] + 1;
    if (h[j] + 1 > H) H = h[j] + 1;
  }
  int64_t* lp = (int64_t*)calloc((size_t)H + 1, sizeof(int64_t));
  for (int64_t j = 0; j < n; ++j) lp[h[j] + 1]++;
  for (int32_t l = 0; l < H; ++l) lp[l + 1] += lp[l];
  int32_t* cols = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
  for (int64_t j = 0; j < n; ++j) fill[j] = 0;
  {
    int64_t* nx = (int64_t*)malloc(sizeof(int64_t) * (size_t)(H + 1));
    for (int32_t l = 0; l <= H; ++l) nx[l] = lp[l];
    for (int64_t j = 0; j < n; ++j) cols[nx[h[j]]++] = (int32_t)j;
    free(nx);
  }
  par_t P;
  memset(&P, 0, sizeof(P));
  P.o = o; P.rp = rp; P.rk = rk; P.rpos = rpos; P.lvl_cols = cols; P.fail = -1;
  pthread_mutex_init(&P.mu, NULL);
  pthread_barrier_init(&P.bar_start, NULL, (unsigned)nthreads);
  pthread_barrier_init(&P.bar_end, NULL, (unsigned)nthreads);
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
  par_arg_t* args = (par_arg_t*)malloc(sizeof(par_arg_t) * (size_t)nthreads);
  for (int t = 0; t < nthreads; ++t) {
    args[t].P = &P;
    args[t].w = (double*)calloc((size_t)n + 1, sizeof(double));
    if (t > 0) pthread_create(&th[t], NULL, par_worker, &args[t]);
  }
  for (int32_t l = 0; l < H; ++l) {
    P.lo = lp[l]; P.hi = lp[l + 1]; P.next = lp[l];
    if (nthreads == 1 || P.hi - P.lo == 1) {   /* a chain column: no hand-off */
      for (int64_t i = P.lo; i < P.hi; ++i) par_column(&P, args[0].w, cols[i]);
      continue;
    }
    pthread_barrier_wait(&P.bar_start);
    for (;;) {
      int64_t i = __atomic_fetch_add(&P.next, 1, __ATOMIC_RELAXED);
      if (i >= P.hi) break;
      par_column(&P, args[0].w, cols[i]);
    }
    pthread_barrier_wait(&P.bar_end);
  }
  P.stop = 1;
  if (nthreads > 1) pthread_barrier_wait(&P.bar_start);
  for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
  for (int t = 0; t < nthreads; ++t) free(args[t].w);
  free(args); free(th);
  pthread_barrier_destroy(&P.bar_start); pthread_barrier_destroy(&P.bar_end); pthread_mutex_destroy(&P.mu);
  free(rp); free(rk); free(rpos); free(fill); free(h); free(lp); free(cols);
  *fail_col = P.fail;
  o->numeric_done = P.fail < 0;
  return P.fail < 0 ? 0 : -3;
}

/* O10: x = P_f^T L^{-T} L^{-1} P_f b */
int orc_solve(const orc_t* o, const double* b, double* x) {
  if (!o->numeric_done) return -7;
  int64_t n = o->n;
  double* y = (double*)malloc(sizeof(double) * (size_t)(n ? n : 1));
  for (int64_t i = 0; i < n; ++i) y[o->perm_final[i]] = b[i];
  const int64_t* Lp = o->Lp; const int32_t* Li = o->Li; const double* Lx = o->Lx;
  for (int64_t j = 0; j < n; ++j) {
    y[j] /= Lx[Lp[j]];
    for (int64_t p = Lp[j] + 1; p < Lp[j + 1]; ++p) y[Li[p]] -= Lx[p] * y[j];
  }
  for (int64_t j = n - 1; j >= 0; --j) {
    for (int64_t p = Lp[j] + 1; p < Lp[j + 1]; ++p) y[j] -= Lx[p] * y[Li[p]];
    y[j] /= Lx[Lp[j]];
  }
  for (int64_t i = 0; i < n; ++i) x[i] = y[o->perm_final[i]];
  free(y);
  return 0;
}

void orc_free(orc_t* o) {
  if (!o) return;
  free(o->post); free(o->parent3); free(o->cc3); free(o->ffirst); free(o->fparent); free(o->fgroup);
  free(o->merge_child); free(o->merge_parent); free(o->merge_cost);
  free(o->perm_final); free(o->o7); free(o->sfirst); free(o->sparent); free(o->rows_ptr); free(o->rows);
  free(o->rel_ptr); free(o->rel_anc); free(o->rel_q0); free(o->rel_off); free(o->relind);
  free(o->blk_ptr); free(o->blk_q); free(o->blk_len); free(o->blk_anc); free(o->blk_relind);
  free(o->parent_final); free(o->cc_final); free(o->Lp); free(o->Li); free(o->Lx);
  free(o->Cp); free(o->Ci); free(o->Cx);
  free(o);
}

/* ---------------- accessors (for the ctypes wrapper) ---------------- */
#define GET(name, type) type orc_get_##name(const orc_t* o) { return o->name; }
GET(n, int64_t) GET(nnzL, int64_t) GET(flops, double) GET(nfund, int32_t) GET(added, int64_t)
GET(nmerges, int32_t) GET(nsuper, int32_t) GET(npairs, int64_t) GET(nblocks, int64_t)
#define PTR(name, type) type* orc_ptr_##name(const orc_t* o) { return o->name; }
PTR(post, int32_t) PTR(parent3, int32_t) PTR(cc3, int32_t) PTR(ffirst, int32_t) PTR(fparent, int32_t)
PTR(fgroup, int32_t) PTR(merge_child, int32_t) PTR(merge_parent, int32_t) PTR(merge_cost, int64_t)
PTR(perm_final, int32_t) PTR(o7, int32_t) PTR(sfirst, int32_t) PTR(sparent, int32_t) PTR(rows_ptr, int64_t)
PTR(rows, int32_t) PTR(rel_ptr, int64_t) PTR(rel_anc, int32_t) PTR(rel_q0, int32_t) PTR(rel_off, int64_t)
PTR(relind, int32_t) PTR(parent_final, int32_t) PTR(cc_final, int32_t) PTR(Lp, int64_t) PTR(Li, int32_t)
PTR(Lx, double) PTR(blk_ptr, int64_t) PTR(blk_q, int32_t) PTR(blk_len, int32_t) PTR(blk_anc, int32_t)
PTR(blk_relind, int32_t)
