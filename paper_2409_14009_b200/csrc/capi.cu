// C ABI (include/spchol.h): handle, device layout in HBM, the level-set launch plan, and the
// factor / solve drivers.  P:n = PAPER.md line n (arXiv 2409.14009).
//
// Device layout (DESIGN.md §Data layout):
//   panels   one FP64 arena; supernode J = column-major m_J x k_J rectangle, ld_J = m_J rounded up
//            to even (16-byte aligned columns for cp.async), offsets int64 ("a supernode
//            is stored in a dense array")
//   amap     int64 destination offset of every stored entry of A (panel init, a1)
//   posmap   int32 per (J, ancestor P) pair and row q of J: position of rows(J)[q] in rows(P)
//            = m_P - 1 - relind(J,P)[q]
//   ucol     per U_J column c: (panel offset of that column inside its ancestor, posmap base)
//   tasks    per launch: batched tile tasks of every supernode of one level (level-set schedule)
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "kernels.cuh"
#include "spchol.h"
#include "symbolic.h"

using namespace spchol;

namespace {
thread_local std::string g_err;
int fail(int code, const std::string& msg) { g_err = msg; return code; }
int cuda_fail(cudaError_t e, const char* where) {
  return fail(e == cudaErrorMemoryAllocation ? SPCHOL_ERR_DEVICE_OOM : SPCHOL_ERR_CUDA,
              std::string(where) + ": " + cudaGetErrorString(e));
}
#define CK(call)                                           \
  do {                                                     \
    cudaError_t e_ = (call);                               \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call);    \
  } while (0)

enum LaunchKind { K_SMALL = 0, K_POTRF = 1, K_TRSM = 2, K_LOCAL = 3, K_SCATTER = 4, K_INIT = 5, K_NKINDS = 6 };
enum OpType { OP_LAUNCH = 0, OP_RECORD = 1, OP_WAIT = 2 };
// One step of the factor's launch plan.  OP_LAUNCH: a batched kernel (kind, tasks [off, off+n)) on
// stream `stream` (0 = critical path: cdiv chain + relind scatter, 1 = trailing updates);
// OP_RECORD / OP_WAIT: event `ev` recorded on / awaited by `stream` (lookahead fork/join).
struct Launch {
  int kind;
  long long off;   // first task
  int n;           // tasks
  double flops, bytes;
  int op = OP_LAUNCH, stream = 0, ev = -1;
  int aux = 0;     // K_SMALL: dynamic shared memory (doubles)
};
template <class T>
cudaError_t dalloc(T** p, size_t count) {
  *p = nullptr;
  if (count == 0) count = 1;
  return cudaMalloc((void**)p, count * sizeof(T));
}
template <class T>
cudaError_t upload(T** p, const std::vector<T>& v) {
  cudaError_t e = dalloc(p, v.size());
  if (e != cudaSuccess) return e;
  if (!v.empty()) e = cudaMemcpy(*p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
  return e;
}
}  // namespace

struct spchol_handle {
  Symbolic S;
  spchol_options opt{};
  int nb = NBMAX;
  static constexpr int OUTER = 4;   // outer block = OUTER inner blocks
  cudaStream_t stream = nullptr, own_stream = nullptr;
  // host plan
  std::vector<SnInfo> sn;
  std::vector<Launch> plan;
  std::vector<GTask> gtasks;
  std::vector<PTask> ptasks;
  std::vector<int> level_sns, level_off;
  std::vector<int> small_sns;           // supernodes handled by the fused small kernel, by level
  std::vector<char> is_small;
  long long panel_doubles = 0;
  std::vector<long long> panel_off;
  double flops_exec = 0, update_entries = 0;
  int max_slots = 0;
  int nslots_total = 0;
  struct SolveStep { int level; long long p0; int np; long long t0; int nt; };
  std::vector<SolveStep> solve_steps;   // per (level, inner block step): POTRF and TRSM task ranges
  std::vector<int> small_level_off;     // small_sns range per level
  int nevents = 0;
  bool no_lookahead = false;     // SPCHOL_NO_LOOKAHEAD=1 (diagnostics)
  std::vector<int> plan_level;   // level of each plan entry (diagnostics)
  // device
  double *d_panels = nullptr, *d_avals = nullptr, *d_linv = nullptr, *d_y = nullptr, *d_y2 = nullptr;
  long long *d_diag_idx = nullptr, *d_amap = nullptr, *d_ucol_base = nullptr, *d_ucol_map = nullptr, *d_rows_ptr = nullptr;
  int *d_small_sns = nullptr, *d_posmap = nullptr, *d_sfirst = nullptr, *d_rows = nullptr, *d_perm = nullptr, *d_level_sns = nullptr;
  SnInfo* d_sn = nullptr;
  GTask* d_gtasks = nullptr;
  PTask* d_ptasks = nullptr;
  unsigned long long* d_fail = nullptr;
  bool values_set = false, factored = false;
  cudaStream_t side_stream = nullptr;           // stream 1 of the plan (trailing updates, low priority)
  cudaStream_t crit_stream = nullptr;           // stream 0 of the plan (cdiv chain, high priority)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  int prio_lo = 0, prio_hi = 0;
  std::vector<cudaEvent_t> plan_events;
  // graph
  cudaGraph_t graph = nullptr, solve_graph = nullptr;
  cudaGraphExec_t gexec = nullptr, solve_gexec = nullptr;
  // timing
  bool timing = false;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  std::vector<std::pair<int, size_t>> pending;  // (plan index, first event)
  long long st_launches[K_NKINDS] = {0};
  double st_ms[K_NKINDS] = {0}, st_flops[K_NKINDS] = {0}, st_bytes[K_NKINDS] = {0};
};

extern "C" void spchol_default_options(spchol_options* o) {
  o->merge_cap = 0.25;
  o->device = 0;
  o->block = 0;
  o->small_max_k = 0;
  o->use_graph = 1;
}

extern "C" const char* spchol_last_error(void) { return g_err.c_str(); }

// ------------------------------------------------------------------------------------- plan
// Lower-triangular tile grid (row tiles starting at rbase, column tiles at cbase, step TILE; a tile
// (r0, s0) is emitted iff r0 < rend, s0 < cend, s0 <= r0) in super-tile order: SUPER x SUPER
// blocks of tiles, row-major inside, so the CTAs in flight share a few operand row blocks in L2
// instead of streaming the whole panel once per row band.
template <class F>
static void for_tiles(int rbase, int rend, int cbase, int cend, F emit) {
  constexpr int SUPER = 8;
  const int nr = rend > rbase ? (rend - rbase + TILE - 1) / TILE : 0;
  const int nc = cend > cbase ? (cend - cbase + TILE - 1) / TILE : 0;
  for (int I = 0; I < nr; I += SUPER)
    for (int Jb = 0; Jb < nc; Jb += SUPER)
      for (int i = I; i < std::min(I + SUPER, nr); ++i)
        for (int j = Jb; j < std::min(Jb + SUPER, nc); ++j) {
          const int r0 = rbase + i * TILE, s0 = cbase + j * TILE;
          if (s0 <= r0) emit(r0, s0);
        }
}

static void build_plan(spchol_handle* h) {
  const Symbolic& S = h->S;
  const int ns = S.nsuper, NB = h->nb, OUTER = spchol_handle::OUTER;
  h->sn.resize(ns);
  h->panel_off.assign(ns + 1, 0);
  for (int J = 0; J < ns; ++J) {
    int k = S.sfirst[J + 1] - S.sfirst[J];
    int m = (int)(S.rows_ptr[J + 1] - S.rows_ptr[J]);
    int ld = m + (m & 1);
    h->sn[J].off = h->panel_off[J];
    h->sn[J].ld = ld; h->sn[J].m = m; h->sn[J].k = k; h->sn[J].ucol = -1;
    h->panel_off[J + 1] = h->panel_off[J] + (long long)ld * k;
    for (int c = 0; c < k; ++c) h->flops_exec += (double)(m - c) * (double)(m - c);
    h->update_entries += 0.5 * (double)(m - k) * (double)(m - k + 1);
  }
  h->panel_doubles = h->panel_off[ns];
  // levels
  h->level_off.assign(S.nlevels + 1, 0);
  for (int J = 0; J < ns; ++J) h->level_off[S.level[J] + 1]++;
  for (int l = 0; l < S.nlevels; ++l) h->level_off[l + 1] += h->level_off[l];
  h->level_sns.assign(ns, 0);
  {
    std::vector<int> nx(h->level_off.begin(), h->level_off.end() - 1);
    for (int J = 0; J < ns; ++J) h->level_sns[nx[S.level[J]]++] = J;
  }
  auto push = [&](int kind, long long off, long long end, double fl, double by) {
    if (end > off) h->plan.push_back(Launch{kind, off, (int)(end - off), fl, by, OP_LAUNCH, 0, -1});
  };
  h->max_slots = 0;
  // fused small-supernode path: k <= small_max_k, m <= 256, m k <= SMALL_MAXELEMS (shared memory)
  const int kmax = h->opt.small_max_k < 0 ? 0 : (h->opt.small_max_k == 0 ? SMALL_MAXK : std::min(h->opt.small_max_k, SMALL_MAXK));
  h->is_small.assign(ns, 0);
  for (int J = 0; J < ns; ++J) {
    const SnInfo& I = h->sn[J];
    h->is_small[J] = I.k <= kmax && I.m <= SMALL_MAXM && (long long)I.m * I.k <= SMALL_MAXELEMS;
  }
  for (int l = 0; l < S.nlevels; ++l) {
    const size_t plan_before = h->plan.size();
    // small supernodes of this level: one launch on stream 1 (independent of the level's big ones)
    {
      long long s0 = (long long)h->small_sns.size();
      h->small_level_off.push_back((int)s0);
      int mx = 0;
      double fsm = 0, bsm = 0;
      for (int x = h->level_off[l]; x < h->level_off[l + 1]; ++x) {
        const int J = h->level_sns[x];
        if (!h->is_small[J]) continue;
        const SnInfo& I = h->sn[J];
        h->small_sns.push_back(J);
        mx = std::max(mx, I.m * I.k);
        const double t = I.m - I.k;
        for (int c = 0; c < I.k; ++c) fsm += (double)(I.m - c) * (double)(I.m - c);
        bsm += 16.0 * I.m * I.k + 16.0 * 0.5 * t * (t + 1);
      }
      long long s1 = (long long)h->small_sns.size();
      if (s1 > s0) {
        const int ev = h->nevents++;
        h->plan.push_back(Launch{0, 0, 0, 0, 0, OP_RECORD, 0, ev});
        h->plan.push_back(Launch{0, 0, 0, 0, 0, OP_WAIT, 1, ev});
        Launch L{K_SMALL, s0, (int)(s1 - s0), fsm, bsm, OP_LAUNCH, 1, -1};
        L.aux = mx;
        h->plan.push_back(L);
      }
    }
    int maxblk = 0;
    for (int x = h->level_off[l]; x < h->level_off[l + 1]; ++x) {
      if (h->is_small[h->level_sns[x]]) continue;
      const SnInfo& I = h->sn[h->level_sns[x]];
      maxblk = std::max(maxblk, (I.k + NB - 1) / NB);
    }
    // two-level blocked right-looking cdiv: inner blocks of NB columns (POTRF + TRSM + update of
    // the rest of the outer block column, K = NB), outer blocks of W = OUTER*NB columns whose
    // trailing update (K = W) is the bulk of the in-panel work.  Lookahead: the outer update of
    // block S is split into NEXT (the columns of outer block S+1, on the critical stream 0) and
    // REST (all later columns, on stream 1), so the cdiv chain of block S+1 (latency-bound POTRF
    // and TRSM launches with few CTAs) overlaps REST(S).  Ordering: REST(S) after the cdiv of
    // block S (event), NEXT(S+1) after REST(S) (same entries), REST(S+1) after REST(S) (stream 1).
    const int W = OUTER * NB;
    int pending_rest_ev = -1;      // event recorded after the latest REST launch on stream 1
    for (int s = 0; s < maxblk; ++s) {
      long long p0 = (long long)h->ptasks.size(), t0 = (long long)h->gtasks.size();
      double fp = 0, ft = 0, fl = 0, bp = 0, bt = 0, bl = 0, fn = 0, bn = 0, fr = 0, br = 0;
      int slot = h->nslots_total;   // every diagonal block keeps its own inverse (reused by the solve)
      std::vector<GTask> local, nxt, rest;
      for (int x = h->level_off[l]; x < h->level_off[l + 1]; ++x) {
        const int J = h->level_sns[x];
        if (h->is_small[J]) continue;
        const SnInfo& I = h->sn[J];
        const int c0 = s * NB;
        if (c0 >= I.k) continue;
        const int nb = std::min(NB, I.k - c0), c1 = c0 + nb;
        const int C0 = (c0 / W) * W, C1 = std::min(C0 + W, I.k);   // enclosing outer block
        h->ptasks.push_back(PTask{J, c0, nb, slot});
        fp += (double)nb * nb * nb / 3.0;
        bp += 16.0 * nb * nb;
        // row tiles start on an even row (16-byte aligned cp.async); rows < c1 are masked (s0 = c1)
        for (int r0 = c1 & ~1; r0 < I.m; r0 += TILE) h->gtasks.push_back(GTask{J, r0, c1, c0, nb, slot});
        ft += (double)(I.m - c1) * nb * nb;
        bt += 16.0 * (double)(I.m - c1) * nb;
        // inner update: columns [c1, C1) of this outer block, K = nb
        for_tiles(c1, I.m, c1, C1, [&](int r0, int s0) { local.push_back(GTask{J, r0, s0, c0, nb, C1}); });
        for (int c = c1; c < C1; ++c) { fl += 2.0 * nb * (double)(I.m - c); bl += 16.0 * (double)(I.m - c); }
        // outer update after the last inner block of the outer block, K = C1 - C0
        if (c1 == C1 && C1 < I.k) {
          const int C2 = std::min(C1 + W, I.k);
          for_tiles(C1, I.m, C1, C2, [&](int r0, int s0) { nxt.push_back(GTask{J, r0, s0, C0, C1 - C0, C2}); });
          for (int c = C1; c < C2; ++c) { fn += 2.0 * (C1 - C0) * (double)(I.m - c); bn += 16.0 * (double)(I.m - c); }
          for_tiles(C2, I.m, C2, I.k, [&](int r0, int s0) { rest.push_back(GTask{J, r0, s0, C0, C1 - C0, I.k}); });
          for (int c = C2; c < I.k; ++c) { fr += 2.0 * (C1 - C0) * (double)(I.m - c); br += 16.0 * (double)(I.m - c); }
        }
        ++slot;
      }
      h->nslots_total = slot;
      long long p1 = (long long)h->ptasks.size(), t1 = (long long)h->gtasks.size();
      if (p1 > p0) h->solve_steps.push_back(spchol_handle::SolveStep{l, p0, (int)(p1 - p0), t0, (int)(t1 - t0)});
      push(K_POTRF, p0, p1, fp, bp);
      push(K_TRSM, t0, t1, ft, bt);
      long long l0 = (long long)h->gtasks.size();
      h->gtasks.insert(h->gtasks.end(), local.begin(), local.end());
      push(K_LOCAL, l0, (long long)h->gtasks.size(), fl, bl);
      if (!rest.empty() && h->no_lookahead) {   // diagnostics: NEXT and REST as one launch, serial
        nxt.insert(nxt.end(), rest.begin(), rest.end());
        fn += fr; bn += br;
        rest.clear();
      }
      if (!rest.empty()) {            // fork REST(S) onto stream 1 after the cdiv of block S
        const int ev = h->nevents++;
        h->plan.push_back(Launch{0, 0, 0, 0, 0, OP_RECORD, 0, ev});
        h->plan.push_back(Launch{0, 0, 0, 0, 0, OP_WAIT, 1, ev});
        long long r0g = (long long)h->gtasks.size();
        h->gtasks.insert(h->gtasks.end(), rest.begin(), rest.end());
        if ((long long)h->gtasks.size() > r0g)
          h->plan.push_back(Launch{K_LOCAL, r0g, (int)((long long)h->gtasks.size() - r0g), fr, br, OP_LAUNCH, 1, -1});
      }
      if (!nxt.empty()) {
        if (pending_rest_ev >= 0) h->plan.push_back(Launch{0, 0, 0, 0, 0, OP_WAIT, 0, pending_rest_ev});
        long long n0 = (long long)h->gtasks.size();
        h->gtasks.insert(h->gtasks.end(), nxt.begin(), nxt.end());
        push(K_LOCAL, n0, (long long)h->gtasks.size(), fn, bn);
      }
      if (!rest.empty()) {
        pending_rest_ev = h->nevents++;
        h->plan.push_back(Launch{0, 0, 0, 0, 0, OP_RECORD, 1, pending_rest_ev});
      }
    }
    bool s1_used = false;
    for (size_t q = plan_before; q < h->plan.size(); ++q) s1_used |= h->plan[q].stream == 1;
    if (s1_used) {  // join stream 1 (small-supernode launch and trailing updates) before the level's scatter
      const int ev = h->nevents++;
      h->plan.push_back(Launch{0, 0, 0, 0, 0, OP_RECORD, 1, ev});
      h->plan.push_back(Launch{0, 0, 0, 0, 0, OP_WAIT, 0, ev});
    }
    (void)pending_rest_ev;
    long long s0g = (long long)h->gtasks.size();
    double fs = 0, bs = 0;
    for (int x = h->level_off[l]; x < h->level_off[l + 1]; ++x) {
      const int J = h->level_sns[x];
      if (h->is_small[J]) continue;
      const SnInfo& I = h->sn[J];
      const int t = I.m - I.k;
      if (t <= 0) continue;
      const int base = I.k & ~1;
      for_tiles(base, I.m, base, I.m, [&](int r0, int c0) { h->gtasks.push_back(GTask{J, r0, c0, 0, 0, 0}); });
      fs += (double)I.k * t * (t + 1);
      bs += 8.0 * (double)t * I.k + 16.0 * 0.5 * t * (t + 1.0);
    }
    push(K_SCATTER, s0g, (long long)h->gtasks.size(), fs, bs);
    h->plan_level.resize(h->plan.size(), l);
  }
  h->small_level_off.push_back((int)h->small_sns.size());
}

static int setup_device(spchol_handle* h) {
  const Symbolic& S = h->S;
  const int ns = S.nsuper;
  // U-column descriptors and posmap
  std::vector<long long> ucb, ucm;
  std::vector<int> posmap(S.relind.size());
  for (long long p = 0; p < (long long)S.rel_anc.size(); ++p) {
    const int P = S.rel_anc[p];
    const long long mP = S.rows_ptr[P + 1] - S.rows_ptr[P];
    for (long long x = S.rel_off[p]; x < S.rel_off[p + 1]; ++x) posmap[x] = (int)(mP - 1 - S.relind[x]);
  }
  for (int J = 0; J < ns; ++J) {
    SnInfo& I = h->sn[J];
    if (I.m - I.k <= 0) continue;
    I.ucol = (int)ucb.size();
    long long pair = S.rel_ptr[J];
    const int* rJ = S.rows.data() + S.rows_ptr[J];
    for (int q = I.k; q < I.m; ++q) {
      while (pair + 1 < S.rel_ptr[J + 1] && S.rel_q0[pair + 1] <= q) ++pair;
      const int P = S.rel_anc[pair];
      ucb.push_back(h->sn[P].off + (long long)(rJ[q] - S.sfirst[P]) * h->sn[P].ld);
      ucm.push_back(S.rel_off[pair] - S.rel_q0[pair]);
    }
  }
  std::vector<long long> amap(S.nnzA);
  for (long long e = 0; e < S.nnzA; ++e) {
    const int c = S.a_col[e], J = S.snode[c];
    amap[e] = h->sn[J].off + (long long)(c - S.sfirst[J]) * h->sn[J].ld + S.a_pos[e];
  }
  CK(cudaSetDevice(h->opt.device));
  CK(kernels_init_attributes());
  CK(cudaStreamCreateWithFlags(&h->own_stream, cudaStreamNonBlocking));
  h->stream = h->own_stream;
  {
    int lo = 0, hi = 0;
    CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));   // numerically lower = higher priority
    h->prio_lo = lo;
    h->prio_hi = hi;
    CK(cudaStreamCreateWithPriority(&h->side_stream, cudaStreamNonBlocking, lo));
    CK(cudaStreamCreateWithPriority(&h->crit_stream, cudaStreamNonBlocking, hi));
    CK(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
  }
  h->plan_events.resize(h->nevents);
  for (auto& e : h->plan_events) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  CK(dalloc(&h->d_panels, (size_t)h->panel_doubles));
  CK(dalloc(&h->d_avals, (size_t)S.nnzA));
  CK(upload(&h->d_amap, amap));
  CK(upload(&h->d_ucol_base, ucb));
  CK(upload(&h->d_ucol_map, ucm));
  CK(upload(&h->d_posmap, posmap));
  CK(upload(&h->d_sn, h->sn));
  CK(upload(&h->d_sfirst, S.sfirst));
  CK(upload(&h->d_gtasks, h->gtasks));
  CK(upload(&h->d_ptasks, h->ptasks));
  CK(dalloc(&h->d_linv, (size_t)std::max(1, h->nslots_total) * NBMAX * NBMAX));
  CK(dalloc(&h->d_fail, 1));
  CK(upload(&h->d_rows_ptr, std::vector<long long>(S.rows_ptr.begin(), S.rows_ptr.end())));
  CK(upload(&h->d_rows, S.rows));
  CK(upload(&h->d_perm, S.perm_final));
  CK(upload(&h->d_level_sns, h->level_sns));
  CK(upload(&h->d_small_sns, h->small_sns));
  CK(dalloc(&h->d_y, (size_t)S.n));
  CK(dalloc(&h->d_y2, (size_t)S.n));
  return SPCHOL_OK;
}

static void free_device(spchol_handle* h) {
  if (h->solve_gexec) cudaGraphExecDestroy(h->solve_gexec);
  if (h->solve_graph) cudaGraphDestroy(h->solve_graph);
  if (h->gexec) cudaGraphExecDestroy(h->gexec);
  if (h->graph) cudaGraphDestroy(h->graph);
  void* ptrs[] = {h->d_small_sns, h->d_diag_idx, h->d_panels, h->d_avals, h->d_linv, h->d_y, h->d_y2, h->d_amap, h->d_ucol_base, h->d_ucol_map,
                  h->d_rows_ptr, h->d_posmap, h->d_sfirst, h->d_rows, h->d_perm, h->d_level_sns, h->d_sn,
                  h->d_gtasks, h->d_ptasks, h->d_fail};
  for (void* p : ptrs) if (p) cudaFree(p);
  for (cudaEvent_t e : h->ev_pool) cudaEventDestroy(e);
  for (cudaEvent_t e : h->plan_events) if (e) cudaEventDestroy(e);
  if (h->side_stream) cudaStreamDestroy(h->side_stream);
  if (h->crit_stream) cudaStreamDestroy(h->crit_stream);
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  if (h->ev_join) cudaEventDestroy(h->ev_join);
  if (h->own_stream) cudaStreamDestroy(h->own_stream);
}

extern "C" int spchol_analyze(int64_t n, const int64_t* colptr, const int32_t* rowidx, const double* values,
                              const int32_t* perm, const spchol_options* opt, spchol_handle** out) {
  if (!out) return fail(SPCHOL_ERR_VALIDATION, "out is NULL");
  *out = nullptr;
  spchol_handle* h = new spchol_handle();
  if (opt) h->opt = *opt; else spchol_default_options(&h->opt);
  if (h->opt.block) {
    if (h->opt.block < 8 || h->opt.block > NBMAX || h->opt.block % 8) { delete h; return fail(SPCHOL_ERR_VALIDATION, "block must be a multiple of 8 in [8, 64]"); }
    h->nb = h->opt.block;
  }
  std::string err;
  int rc = analyze_symbolic(n, colptr, rowidx, perm, h->opt.merge_cap, h->S, err);
  if (rc != SPCHOL_OK) { delete h; return fail(rc, err); }
  if (const char* e = getenv("SPCHOL_NO_LOOKAHEAD")) h->no_lookahead = atoi(e) != 0;
  build_plan(h);
  if (h->opt.device < 0) { *out = h; return SPCHOL_OK; }   // host-only analysis (no device state)
  rc = setup_device(h);
  if (rc != SPCHOL_OK) { free_device(h); delete h; return rc; }
  if (values) {
    rc = spchol_set_values(h, values);
    if (rc != SPCHOL_OK) { free_device(h); delete h; return rc; }
  }
  *out = h;
  return SPCHOL_OK;
}

static bool host_only(const spchol_handle* h) { return h->opt.device < 0; }

extern "C" int spchol_set_values(spchol_handle* h, const double* values) {
  if (!h || !values) return fail(SPCHOL_ERR_VALIDATION, "NULL handle or values");
  if (host_only(h)) return fail(SPCHOL_ERR_STATE, "host-only handle (device < 0)");
  CK(cudaSetDevice(h->opt.device));
  CK(cudaMemcpyAsync(h->d_avals, values, sizeof(double) * (size_t)h->S.nnzA, cudaMemcpyHostToDevice, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  h->values_set = true;
  h->factored = false;
  return SPCHOL_OK;
}

extern "C" int spchol_set_values_device(spchol_handle* h, const double* d_values) {
  if (!h || !d_values) return fail(SPCHOL_ERR_VALIDATION, "NULL handle or values");
  if (host_only(h)) return fail(SPCHOL_ERR_STATE, "host-only handle (device < 0)");
  CK(cudaSetDevice(h->opt.device));
  CK(cudaMemcpyAsync(h->d_avals, d_values, sizeof(double) * (size_t)h->S.nnzA, cudaMemcpyDeviceToDevice, h->stream));
  h->values_set = true;
  h->factored = false;
  return SPCHOL_OK;
}

extern "C" int spchol_set_stream(spchol_handle* h, void* stream) {
  if (!h) return fail(SPCHOL_ERR_VALIDATION, "NULL handle");
  h->stream = stream ? (cudaStream_t)stream : h->own_stream;
  return SPCHOL_OK;
}

// Enqueue the whole factorization on st (no host synchronization).
static int enqueue_factor(spchol_handle* h, cudaStream_t st) {
  const Symbolic& S = h->S;
  auto tstart = [&](int idx) -> size_t {
    if (!h->timing) return 0;
    while (h->ev_used + 2 > h->ev_pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      h->ev_pool.push_back(e);
    }
    size_t i = h->ev_used;
    h->ev_used += 2;
    cudaEventRecord(h->ev_pool[i], st);
    h->pending.push_back({idx, i});
    return i;
  };
  auto tstop = [&](size_t i) { if (h->timing) cudaEventRecord(h->ev_pool[i + 1], st); };
  CK(cudaMemsetAsync(h->d_fail, 0xFF, sizeof(unsigned long long), st));
  size_t ti = tstart(-1);
  CK(cudaMemsetAsync(h->d_panels, 0, sizeof(double) * (size_t)std::max(1LL, h->panel_doubles), st));
  launch_init(h->d_avals, h->d_amap, S.nnzA, h->d_panels, st);
  tstop(ti);
  // The plan's stream 0 (critical path) runs on a high-priority internal stream so its few-CTA
  // cdiv launches are scheduled ahead of the trailing-update CTAs of stream 1 (low priority).
  // Both fork from st and join back into it (required under graph capture).  With kernel
  // timing enabled everything runs serialized on st.
  const bool multi = !h->timing;
  cudaStream_t s0 = multi ? h->crit_stream : st;
  cudaStream_t s1 = multi ? h->side_stream : st;
  if (multi) {
    CK(cudaEventRecord(h->ev_fork, st));
    CK(cudaStreamWaitEvent(s0, h->ev_fork, 0));
  }
  for (size_t i = 0; i < h->plan.size(); ++i) {
    const Launch& L = h->plan[i];
    cudaStream_t ls = L.stream == 1 ? s1 : s0;
    if (L.op == OP_RECORD) {
      if (multi) CK(cudaEventRecord(h->plan_events[L.ev], ls));
      continue;
    }
    if (L.op == OP_WAIT) {
      if (multi) CK(cudaStreamWaitEvent(ls, h->plan_events[L.ev], 0));
      continue;
    }
    ti = tstart((int)i);
    const int prio = multi ? (L.stream == 1 ? h->prio_lo : h->prio_hi) : 0;
    switch (L.kind) {
      case K_SMALL:
        launch_small(h->d_small_sns + L.off, L.n, h->d_sn, h->d_sfirst, h->d_panels, h->d_ucol_base, h->d_ucol_map,
                     h->d_posmap, h->d_fail, L.aux, ls, prio);
        break;
      case K_POTRF:
        launch_potrf(h->d_ptasks + L.off, L.n, h->d_sn, h->d_sfirst, h->d_panels, h->d_linv, h->d_fail, ls, prio);
        break;
      case K_TRSM:
        launch_gemm(MODE_TRSM, h->d_gtasks + L.off, L.n, h->d_sn, h->d_panels, h->d_linv, h->d_ucol_base, h->d_ucol_map, h->d_posmap, ls, prio);
        break;
      case K_LOCAL:
        launch_gemm(MODE_LOCAL, h->d_gtasks + L.off, L.n, h->d_sn, h->d_panels, h->d_linv, h->d_ucol_base, h->d_ucol_map, h->d_posmap, ls, prio);
        break;
      case K_SCATTER:
        launch_gemm(MODE_SCATTER, h->d_gtasks + L.off, L.n, h->d_sn, h->d_panels, h->d_linv, h->d_ucol_base, h->d_ucol_map, h->d_posmap, ls, prio);
        break;
    }
    tstop(ti);
  }
  if (multi) {
    CK(cudaEventRecord(h->ev_join, s0));
    CK(cudaStreamWaitEvent(st, h->ev_join, 0));
  }
  CK(cudaGetLastError());
  return SPCHOL_OK;
}

extern "C" int spchol_factor_async(spchol_handle* h) {
  if (!h) return fail(SPCHOL_ERR_VALIDATION, "NULL handle");
  if (host_only(h)) return fail(SPCHOL_ERR_STATE, "host-only handle (device < 0)");
  if (!h->values_set) return fail(SPCHOL_ERR_STATE, "values not set");
  CK(cudaSetDevice(h->opt.device));
  h->factored = false;
  if (h->opt.use_graph && !h->timing) {
    if (!h->gexec) {
      cudaStream_t cs = h->own_stream;
      CK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
      int rc = enqueue_factor(h, cs);
      cudaGraph_t g = nullptr;
      cudaError_t e = cudaStreamEndCapture(cs, &g);
      if (rc != SPCHOL_OK) { if (g) cudaGraphDestroy(g); return rc; }
      if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture");
      h->graph = g;
      CK(cudaGraphInstantiateWithFlags(&h->gexec, g, cudaGraphInstantiateFlagUseNodePriority));  // honour per-node priorities
    }
    CK(cudaGraphLaunch(h->gexec, h->stream));
    return SPCHOL_OK;
  }
  return enqueue_factor(h, h->stream);
}

extern "C" int spchol_factor_status(spchol_handle* h, int64_t* fail_col, int64_t* fail_col_orig) {
  if (!h) return fail(SPCHOL_ERR_VALIDATION, "NULL handle");
  if (host_only(h)) return fail(SPCHOL_ERR_STATE, "host-only handle (device < 0)");
  CK(cudaSetDevice(h->opt.device));
  CK(cudaStreamSynchronize(h->stream));
  unsigned long long f = 0;
  CK(cudaMemcpy(&f, h->d_fail, sizeof(f), cudaMemcpyDeviceToHost));
  int64_t fc = f == ~0ULL ? -1 : (int64_t)f;
  if (fail_col) *fail_col = fc;
  if (fail_col_orig) *fail_col_orig = fc < 0 ? -1 : h->S.iperm_final[fc];
  if (fc >= 0) {
    h->factored = false;
    return fail(SPCHOL_ERR_NOT_SPD, "matrix is not positive definite: pivot <= 0 at final column " + std::to_string(fc));
  }
  h->factored = true;
  return SPCHOL_OK;
}

extern "C" int spchol_factor(spchol_handle* h, int64_t* fail_col, int64_t* fail_col_orig) {
  int rc = spchol_factor_async(h);
  if (rc != SPCHOL_OK) return rc;
  return spchol_factor_status(h, fail_col, fail_col_orig);
}

// Supernodal triangular solves: y = P_f b; forward L y' = y level by level (leaves first),
// backward L^T z = y' (root first); x = P_f^T z.  Small supernodes: one CTA each (column sweep in
// the CTA).  Large supernodes: per inner 64-column block b, y_b := X_bb y_b with the diagonal-block
// inverse kept from the factor, then the rows below are updated by a row-tiled block GEMV (RED into
// y); backward in reverse with the transposed operations.
static int enqueue_solve(spchol_handle* h, const double* d_b, double* d_x, cudaStream_t st) {
  const Symbolic& S = h->S;
  launch_permute(h->d_perm, d_b, h->d_y, S.n, 0, st);
  std::vector<std::pair<size_t, size_t>> lvl_steps(S.nlevels, {0, 0});
  for (size_t q = 0; q < h->solve_steps.size(); ++q) {
    auto& r = lvl_steps[h->solve_steps[q].level];
    if (r.second == 0) r.first = q;
    r.second = q + 1;
  }
  for (int l = 0; l < S.nlevels; ++l) {
    launch_solve_fwd(h->d_small_sns + h->small_level_off[l], h->small_level_off[l + 1] - h->small_level_off[l], h->d_sn,
                     h->d_sfirst, h->d_rows_ptr, h->d_rows, h->d_panels, h->d_y, st);
    for (size_t q = lvl_steps[l].first; q < lvl_steps[l].second; ++q) {
      const auto& T = h->solve_steps[q];
      launch_solve_diag(h->d_ptasks + T.p0, T.np, h->d_sfirst, h->d_linv, h->d_y, 0, st);
      launch_solve_upd(h->d_gtasks + T.t0, T.nt, h->d_sn, h->d_sfirst, h->d_rows_ptr, h->d_rows, h->d_panels, h->d_y, 0, st);
    }
  }
  for (int l = S.nlevels - 1; l >= 0; --l) {
    for (size_t q = lvl_steps[l].second; q > lvl_steps[l].first; --q) {
      const auto& T = h->solve_steps[q - 1];
      launch_solve_upd(h->d_gtasks + T.t0, T.nt, h->d_sn, h->d_sfirst, h->d_rows_ptr, h->d_rows, h->d_panels, h->d_y, 1, st);
      launch_solve_diag(h->d_ptasks + T.p0, T.np, h->d_sfirst, h->d_linv, h->d_y, 1, st);
    }
    launch_solve_bwd(h->d_small_sns + h->small_level_off[l], h->small_level_off[l + 1] - h->small_level_off[l], h->d_sn,
                     h->d_sfirst, h->d_rows_ptr, h->d_rows, h->d_panels, h->d_y, st);
  }
  launch_permute(h->d_perm, h->d_y, d_x, S.n, 1, st);
  CK(cudaGetLastError());
  return SPCHOL_OK;
}

// One solve of the internal buffer d_y2 in place, captured in a CUDA graph on first use.
static int run_solve_y2(spchol_handle* h) {
  if (!h->opt.use_graph) return enqueue_solve(h, h->d_y2, h->d_y2, h->stream);
  if (!h->solve_gexec) {
    cudaStream_t cs = h->own_stream;
    CK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    int rc = enqueue_solve(h, h->d_y2, h->d_y2, cs);
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamEndCapture(cs, &g);
    if (rc != SPCHOL_OK) { if (g) cudaGraphDestroy(g); return rc; }
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture(solve)");
    h->solve_graph = g;
    CK(cudaGraphInstantiateWithFlags(&h->solve_gexec, g, 0));
  }
  CK(cudaGraphLaunch(h->solve_gexec, h->stream));
  return SPCHOL_OK;
}

extern "C" int spchol_solve_device(spchol_handle* h, const double* d_b, double* d_x, int32_t nrhs, int64_t ld) {
  if (!h) return fail(SPCHOL_ERR_VALIDATION, "NULL handle");
  if (host_only(h) || !h->factored) return fail(SPCHOL_ERR_STATE, "solve before a successful factor");
  if (nrhs < 1 || ld < h->S.n) return fail(SPCHOL_ERR_DIMENSION, "nrhs < 1 or ld < n");
  CK(cudaSetDevice(h->opt.device));
  const size_t nbytes = sizeof(double) * (size_t)h->S.n;
  for (int r = 0; r < nrhs; ++r) {
    CK(cudaMemcpyAsync(h->d_y2, d_b + (size_t)r * ld, nbytes, cudaMemcpyDeviceToDevice, h->stream));
    int rc = run_solve_y2(h);
    if (rc != SPCHOL_OK) return rc;
    CK(cudaMemcpyAsync(d_x + (size_t)r * ld, h->d_y2, nbytes, cudaMemcpyDeviceToDevice, h->stream));
  }
  return SPCHOL_OK;
}

extern "C" int spchol_solve(spchol_handle* h, const double* b, double* x, int32_t nrhs, int64_t ld) {
  if (!h) return fail(SPCHOL_ERR_VALIDATION, "NULL handle");
  if (host_only(h) || !h->factored) return fail(SPCHOL_ERR_STATE, "solve before a successful factor");
  if (nrhs < 1 || ld < h->S.n) return fail(SPCHOL_ERR_DIMENSION, "nrhs < 1 or ld < n");
  CK(cudaSetDevice(h->opt.device));
  const size_t nbytes = sizeof(double) * (size_t)h->S.n;
  for (int r = 0; r < nrhs; ++r) {
    CK(cudaMemcpyAsync(h->d_y2, b + (size_t)r * ld, nbytes, cudaMemcpyHostToDevice, h->stream));
    int rc = run_solve_y2(h);
    if (rc != SPCHOL_OK) return rc;
    CK(cudaMemcpyAsync(x + (size_t)r * ld, h->d_y2, nbytes, cudaMemcpyDeviceToHost, h->stream));
  }
  CK(cudaStreamSynchronize(h->stream));
  return SPCHOL_OK;
}

extern "C" int spchol_query(const spchol_handle* h, int key, int64_t* value) {
  if (!h || !value) return fail(SPCHOL_ERR_VALIDATION, "NULL argument");
  const Symbolic& S = h->S;
  switch (key) {
    case SPCHOL_Q_N: *value = S.n; break;
    case SPCHOL_Q_NNZ_A: *value = S.nnzA; break;
    case SPCHOL_Q_NNZ_L: *value = S.nnzL; break;
    case SPCHOL_Q_NFUND: *value = (int64_t)S.ffirst.size() - 1; break;
    case SPCHOL_Q_NSUPER: *value = S.nsuper; break;
    case SPCHOL_Q_ADDED: *value = S.added; break;
    case SPCHOL_Q_NLEVELS: *value = S.nlevels; break;
    case SPCHOL_Q_ROWS_LEN: *value = (int64_t)S.rows.size(); break;
    case SPCHOL_Q_NPAIRS: *value = (int64_t)S.rel_anc.size(); break;
    case SPCHOL_Q_RELIND_LEN: *value = (int64_t)S.relind.size(); break;
    case SPCHOL_Q_PANEL_DOUBLES: *value = h->panel_doubles; break;
    case SPCHOL_Q_NMERGES: *value = S.nmerges; break;
    case SPCHOL_Q_FLOPS_EXACT: *value = (int64_t)S.flops_exact; break;
    case SPCHOL_Q_FLOPS_EXEC: *value = (int64_t)h->flops_exec; break;
    case SPCHOL_Q_LAUNCHES: {
      int64_t nl = 1;
      for (const Launch& L : h->plan) nl += L.op == OP_LAUNCH;
      *value = nl;
      break;
    }
    case SPCHOL_Q_UPDATE_ENTRIES: *value = (int64_t)h->update_entries; break;
    default: return fail(SPCHOL_ERR_VALIDATION, "unknown query key");
  }
  return SPCHOL_OK;
}

template <class T>
static void cp(T* dst, const std::vector<T>& v) { if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(T)); }

extern "C" int spchol_export_symbolic(const spchol_handle* h, int32_t* post, int32_t* parent3, int32_t* cc3,
                                      int32_t* ffirst, int32_t* fgroup, int32_t* perm_final, int32_t* sfirst,
                                      int32_t* sparent, int64_t* rows_ptr, int32_t* rows, int64_t* rel_ptr,
                                      int32_t* rel_anc, int32_t* rel_q0, int64_t* rel_off, int32_t* relind,
                                      int32_t* parent_final, int32_t* cc_final, int32_t* level) {
  if (!h) return fail(SPCHOL_ERR_VALIDATION, "NULL handle");
  const Symbolic& S = h->S;
  cp(post, S.post); cp(parent3, S.parent3); cp(cc3, S.cc3); cp(ffirst, S.ffirst); cp(fgroup, S.fgroup);
  cp(perm_final, S.perm_final); cp(sfirst, S.sfirst); cp(sparent, S.sparent);
  cp<int64_t>(rows_ptr, S.rows_ptr); cp(rows, S.rows); cp<int64_t>(rel_ptr, S.rel_ptr); cp(rel_anc, S.rel_anc);
  cp(rel_q0, S.rel_q0); cp<int64_t>(rel_off, S.rel_off); cp(relind, S.relind); cp(parent_final, S.parent_final);
  cp(cc_final, S.cc_final); cp(level, S.level);
  return SPCHOL_OK;
}

extern "C" int spchol_export_panels(const spchol_handle* h, int64_t* panel_off, int32_t* ld, double* panels) {
  if (!h) return fail(SPCHOL_ERR_VALIDATION, "NULL handle");
  if (host_only(h) && panels) return fail(SPCHOL_ERR_STATE, "host-only handle (device < 0)");
  if (host_only(h)) {
    if (panel_off) for (size_t J = 0; J < h->panel_off.size(); ++J) panel_off[J] = h->panel_off[J];
    if (ld) for (size_t J = 0; J < h->sn.size(); ++J) ld[J] = h->sn[J].ld;
    return SPCHOL_OK;
  }
  CK(cudaSetDevice(h->opt.device));
  CK(cudaStreamSynchronize(h->stream));
  if (panel_off) for (size_t J = 0; J < h->panel_off.size(); ++J) panel_off[J] = h->panel_off[J];
  if (ld) for (size_t J = 0; J < h->sn.size(); ++J) ld[J] = h->sn[J].ld;
  if (panels && h->panel_doubles > 0)
    CK(cudaMemcpy(panels, h->d_panels, sizeof(double) * (size_t)h->panel_doubles, cudaMemcpyDeviceToHost));
  return SPCHOL_OK;
}

extern "C" int spchol_export_panel(const spchol_handle* h, int32_t J, double* out) {
  if (!h || !out) return fail(SPCHOL_ERR_VALIDATION, "NULL argument");
  if (host_only(h)) return fail(SPCHOL_ERR_STATE, "host-only handle (device < 0)");
  if (J < 0 || J >= h->S.nsuper) return fail(SPCHOL_ERR_DIMENSION, "supernode index out of range");
  CK(cudaSetDevice(h->opt.device));
  CK(cudaStreamSynchronize(h->stream));
  const size_t cnt = (size_t)(h->panel_off[J + 1] - h->panel_off[J]);
  if (cnt) CK(cudaMemcpy(out, h->d_panels + h->panel_off[J], sizeof(double) * cnt, cudaMemcpyDeviceToHost));
  return SPCHOL_OK;
}

extern "C" int spchol_export_diagonal(spchol_handle* h, double* diag) {
  if (!h || !diag) return fail(SPCHOL_ERR_VALIDATION, "NULL argument");
  if (host_only(h)) return fail(SPCHOL_ERR_STATE, "host-only handle (device < 0)");
  CK(cudaSetDevice(h->opt.device));
  const Symbolic& S = h->S;
  if (!h->d_diag_idx) {
    std::vector<long long> idx(S.n);
    for (int J = 0; J < S.nsuper; ++J)
      for (int c = 0; c < h->sn[J].k; ++c) idx[S.sfirst[J] + c] = h->sn[J].off + (long long)c * h->sn[J].ld + c;
    CK(upload(&h->d_diag_idx, idx));
  }
  launch_gather(h->d_panels, h->d_diag_idx, h->d_y, S.n, h->stream);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(diag, h->d_y, sizeof(double) * (size_t)S.n, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  return SPCHOL_OK;
}

extern "C" int spchol_kernel_trace(spchol_handle* h, int64_t cap, int64_t* count, int32_t* kinds, int32_t* levels,
                                   int32_t* ntasks, double* ms) {
  if (!h || !count) return fail(SPCHOL_ERR_VALIDATION, "NULL argument");
  if (host_only(h)) return fail(SPCHOL_ERR_STATE, "host-only handle (device < 0)");
  CK(cudaSetDevice(h->opt.device));
  CK(cudaStreamSynchronize(h->stream));
  int64_t c = 0;
  for (auto& pr : h->pending) {
    if (c < cap) {
      float t = 0;
      cudaEventElapsedTime(&t, h->ev_pool[pr.second], h->ev_pool[pr.second + 1]);
      if (kinds) kinds[c] = pr.first < 0 ? K_INIT : h->plan[pr.first].kind;
      if (levels) levels[c] = pr.first < 0 ? -1 : h->plan_level[pr.first];
      if (ntasks) ntasks[c] = pr.first < 0 ? 0 : h->plan[pr.first].n;
      if (ms) ms[c] = t;
    }
    ++c;
  }
  *count = c;
  return SPCHOL_OK;
}

extern "C" int spchol_enable_kernel_timing(spchol_handle* h, int enable) {
  if (!h) return fail(SPCHOL_ERR_VALIDATION, "NULL handle");
  h->timing = enable != 0;
  for (int k = 0; k < K_NKINDS; ++k) { h->st_launches[k] = 0; h->st_ms[k] = h->st_flops[k] = h->st_bytes[k] = 0.0; }
  h->pending.clear();
  h->ev_used = 0;
  return SPCHOL_OK;
}

extern "C" int spchol_kernel_stats(spchol_handle* h, int kind, int64_t* launches, double* ms, double* flops,
                                   double* bytes) {
  if (!h) return fail(SPCHOL_ERR_VALIDATION, "NULL handle");
  if (kind < 0 || kind >= K_NKINDS) return fail(SPCHOL_ERR_VALIDATION, "bad kernel kind");
  if (host_only(h)) return fail(SPCHOL_ERR_STATE, "host-only handle (device < 0)");
  CK(cudaSetDevice(h->opt.device));
  CK(cudaStreamSynchronize(h->stream));
  for (auto& pr : h->pending) {
    float t = 0;
    cudaEventElapsedTime(&t, h->ev_pool[pr.second], h->ev_pool[pr.second + 1]);
    int kd = pr.first < 0 ? K_INIT : h->plan[pr.first].kind;
    h->st_launches[kd] += 1;
    h->st_ms[kd] += t;
    if (pr.first < 0) {
      h->st_bytes[kd] += 8.0 * (double)h->panel_doubles + 16.0 * (double)h->S.nnzA + 8.0 * h->S.nnzA;
    } else {
      h->st_flops[kd] += h->plan[pr.first].flops;
      h->st_bytes[kd] += h->plan[pr.first].bytes;
    }
  }
  h->pending.clear();
  h->ev_used = 0;
  if (launches) *launches = h->st_launches[kind];
  if (ms) *ms = h->st_ms[kind];
  if (flops) *flops = h->st_flops[kind];
  if (bytes) *bytes = h->st_bytes[kind];
  return SPCHOL_OK;
}

extern "C" void spchol_destroy(spchol_handle* h) {
  if (!h) return;
  if (!host_only(h)) {
    cudaSetDevice(h->opt.device);
    free_device(h);
  }
  delete h;
}
