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
#include <dlfcn.h>

#include <algorithm>
#include <array>
#include <climits>
#include <cstdint>
#include <mutex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <cudaTypedefs.h>
#include <nvtx3/nvToolsExt.h>

#include "handle.h"

using namespace spchol;
namespace spchol {
void proportional_map(const Symbolic& S, const std::vector<double>& work, int world, std::vector<int>& owner,
                      std::vector<int>* top_lo = nullptr, std::vector<int>* top_hi = nullptr);
void assign_top_owners(const std::vector<double>& work, const std::vector<int>& owner, const std::vector<int>& lo,
                       const std::vector<int>& hi, const std::vector<int>& level, int world,
                       std::vector<int>& top_owner);

namespace {
thread_local std::string g_err;
}
// NVTX ranges (SURVEY §5 tracing): analyze, factor (enqueue or graph launch), each level's plan
// range when enqueued eagerly, solve, exchanges; visible in Nsight Systems / ncu --nvtx.
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
};
int fail(int code, const std::string& msg) { g_err = msg; return code; }
int cuda_fail(cudaError_t e, const char* where) {
  return fail(e == cudaErrorMemoryAllocation ? SPCHOL_ERR_DEVICE_OOM : SPCHOL_ERR_CUDA,
              std::string(where) + ": " + cudaGetErrorString(e));
}
thread_local size_t g_dev_bytes = 0;

// ------------------------------------------------------------------------------------- NCCL
NcclApi g_nccl;
namespace {
std::mutex g_nccl_mu;   // handles (and the tests' rank threads) may attach concurrently
}
// Resolves every symbol into a local table first and publishes it (g_nccl.so last) under the lock.
bool nccl_load(std::string& err) {
  std::lock_guard<std::mutex> lock(g_nccl_mu);
  if (g_nccl.so) return true;
  NcclApi api;
  // SPCHOL_NCCL_LIB: another NCCL build, or the tests' single-GPU stand-in (tests/mock_nccl)
  const char* alt = getenv("SPCHOL_NCCL_LIB");
  void* so = dlopen(alt && *alt ? alt : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!so) so = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!so) { err = std::string("cannot load NCCL: ") + dlerror(); return false; }
  api.getid = (nccl_getid_t)dlsym(so, "ncclGetUniqueId");
  api.init = (nccl_init_t)dlsym(so, "ncclCommInitRank");
  api.allreduce = (nccl_allreduce_t)dlsym(so, "ncclAllReduce");
  api.reduce = (nccl_reduce_t)dlsym(so, "ncclReduce");
  api.send = (nccl_p2p_t)dlsym(so, "ncclSend");
  api.bcast = (nccl_bcast_t)dlsym(so, "ncclBroadcast");
  api.split = (nccl_split_t)dlsym(so, "ncclCommSplit");
  api.recv = (nccl_p2p_t)dlsym(so, "ncclRecv");
  api.group_start = (nccl_group_t)dlsym(so, "ncclGroupStart");
  api.group_end = (nccl_group_t)dlsym(so, "ncclGroupEnd");
  api.destroy = (nccl_destroy_t)dlsym(so, "ncclCommDestroy");
  api.errstr = (nccl_errstr_t)dlsym(so, "ncclGetErrorString");
  // the tests' stand-in blocks the host inside every call, so its calls cannot be graph-captured
  api.capturable = dlsym(so, "spcholMockNcclBlocking") == nullptr;
  if (!api.getid || !api.init || !api.allreduce || !api.reduce || !api.send || !api.recv || !api.bcast || !api.split || !api.group_start ||
      !api.group_end || !api.destroy) { err = "NCCL symbols missing"; return false; }
  api.so = so;
  g_nccl = api;
  return true;
}
int nccl_fail(int r, const char* where) {
  return fail(SPCHOL_ERR_NCCL, std::string(where) + ": " + (g_nccl.errstr ? g_nccl.errstr(r) : "nccl error"));
}
}  // namespace spchol

extern "C" void spchol_default_options(spchol_options* o) {
  o->merge_cap = 0.25;
  o->device = 0;
  o->block = 0;
  o->small_max_k = 0;
  o->use_graph = 1;
  o->dist_rank = 0;
  o->dist_world = 1;
  o->subtree_streams = 0;
  o->update_mode = 0;
  o->deterministic = 0;
  o->partition_refinement = 0;
  o->device_mem_cap = 0;
}

extern "C" const char* spchol_last_error(void) { return g_err.c_str(); }

// ------------------------------------------------------------------------------------- plan
// Lower-triangular tile grid (row tiles starting at rbase, column tiles at cbase, step TILE; a tile
// (r0, s0) is emitted iff r0 < rend, s0 < cend, s0 <= r0) in super-tile order: SUPER x SUPER
// blocks of tiles, row-major inside, so the CTAs in flight share a few operand row blocks in L2
// instead of streaming the whole panel once per row band.
template <class F>
static void for_tiles(int rbase, int rend, int cbase, int cend, F emit) {
#ifndef SPCHOL_SUPER
#define SPCHOL_SUPER 8
#endif
  constexpr int SUPER = SPCHOL_SUPER;
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

// The NCCL communicator of top supernode J's rank group (ranks lo..hi-1 as 0..hi-lo-1): the world
// communicator when the group is everyone, else the one ncclCommSplit made at attach time.
void* spchol::group_comm(const spchol_handle* h, int J) {
  if (h->grp_hi[J] - h->grp_lo[J] == h->world) return h->nccl_comm;
  for (size_t i = 0; i < h->grp_keys.size(); ++i)
    if (h->grp_keys[i][0] == h->grp_lo[J] && h->grp_keys[i][1] == h->grp_hi[J]) return h->grp_comms[i];
  return nullptr;
}

// Deterministic mode (reading C-7): greedy column-conflict colouring of the supernodes Js (ascending
// order): J takes the lowest colour none of whose members shares an update column (R_J) with it.
// Within a colour no two supernodes update one ancestor entry, so their scatter needs no RED.
static int colour_supernodes(const spchol_handle* h, const std::vector<int>& Js, std::vector<int>& colour) {
  const Symbolic& S = h->S;
  static thread_local std::vector<std::vector<char>> used;   // used[c][col]
  colour.assign(Js.size(), 0);
  int ncol = 0;
  for (size_t x = 0; x < Js.size(); ++x) {
    const int J = Js[x];
    const long long b = S.rows_ptr[J] + h->sn[J].k, e = S.rows_ptr[J + 1];
    int c = 0;
    for (;; ++c) {
      if (c == (int)used.size()) used.emplace_back();
      if (used[c].size() < (size_t)S.n) used[c].assign(S.n, 0);
      bool clash = false;
      for (long long q = b; q < e && !clash; ++q) clash = used[c][S.rows[q]];
      if (!clash) break;
    }
    for (long long q = b; q < e; ++q) used[c][S.rows[q]] = 1;
    colour[x] = c;
    ncol = std::max(ncol, c + 1);
  }
  for (size_t x = 0; x < Js.size(); ++x) {   // reset the marks for the next level
    const int J = Js[x];
    for (long long q = S.rows_ptr[J] + h->sn[J].k; q < S.rows_ptr[J + 1]; ++q) used[colour[x]][S.rows[q]] = 0;
  }
  return std::max(ncol, 1);
}

// Appends, level by level, the launches for the supernodes J with active(J).  record_solve: also
// record the solve's step structure (only for the whole-tree plan).  top_markers (multi-GPU phase
// C of rank h->rank): distributed top supernodes (top_dist) take part on every rank of their group —
// cdiv tasks of the column blocks the rank owns, one OP_BCAST marker per finished column block (on
// every rank, so all plans hold the same marker sequence), and the rank's partial U_J (its own block
// columns' share of the K sum, MODE_SCATTER_KS); after each level with update blocks, an OP_EXCHANGE.
template <class Active>
static void append_levels(spchol_handle* h, Active active, bool record_solve, int SB = 0, bool top_markers = false) {
  const Symbolic& S = h->S;
  const int NB = h->nb, OUTER = h->outer;
  auto push = [&](int kind, long long off, long long end, double fl, double by) {
    if (end > off) h->plan.push_back(Launch{kind, off, (int)(end - off), fl, by, OP_LAUNCH, SB, -1});
  };
  const int lmax = h->max_level >= 0 ? std::min(S.nlevels, h->max_level + 1) : S.nlevels;
  for (int l = 0; l < lmax; ++l) {
    const size_t plan_before = h->plan.size();
    // small supernodes of this level: launches on stream 1 (independent of the level's big ones),
    // bucketed by panel size so that each launch's shared memory (sized by its largest panel)
    // lets as many CTAs as possible be resident
    {
      if (record_solve) h->small_level_off.push_back((int)h->small_sns.size());
      // warp kernel (m <= 128): one launch per rows-per-lane class; CTA kernel (m > 128, or
      // SPCHOL_SMALL_WARP=0): buckets by m k
      static const int bucket_max[] = {256, 1024, 4096, SMALL_MAXELEMS};
      auto bucket = [&](const SnInfo& I) {
        // warp kernel: by rows per lane and by k (the launch's shared memory follows its largest k)
        if (h->small_warp && I.m <= h->small_warp_maxm)
          return 3 * (I.k <= 16 ? 0 : I.k <= 32 ? 1 : 2) + (I.m <= 32 ? 0 : (I.m <= 64 ? 1 : 2));
        const int mk = I.m * I.k;
        return 9 + (mk <= 256 ? 0 : mk <= 1024 ? 1 : mk <= 4096 ? 2 : 3);
      };
      (void)bucket_max;
      bool forked = false;
      std::vector<int> sm, scol;
      for (int x = h->level_off[l]; x < h->level_off[l + 1]; ++x)
        if (h->is_small[h->level_sns[x]] && active(h->level_sns[x])) sm.push_back(h->level_sns[x]);
      const int nsc = h->opt.deterministic ? colour_supernodes(h, sm, scol) : 1;
      if (!h->opt.deterministic) scol.assign(sm.size(), 0);
      for (int col = 0; col < nsc; ++col)
      for (int bk = 0; bk < 13; ++bk) {
        long long s0 = (long long)h->small_sns.size();
        int mx = 0, mxm = 0, mxk = 0;
        double fsm = 0, bsm = 0;
        for (size_t x = 0; x < sm.size(); ++x) {
          const int J = sm[x];
          if (scol[x] != col) continue;
          const SnInfo& I = h->sn[J];
          const int mk = I.m * I.k;
          if (bucket(I) != bk) continue;
          h->small_sns.push_back(J);
          mx = std::max(mx, bk < 9 ? mk : small_cta_smem(I.m, I.k));
          mxm = std::max(mxm, I.m);
          mxk = std::max(mxk, I.k);
          const double t = I.m - I.k;
          for (int c = 0; c < I.k; ++c) fsm += (double)(I.m - c) * (double)(I.m - c);
          bsm += 16.0 * I.m * I.k + 16.0 * 0.5 * t * (t + 1);
        }
        long long s1 = (long long)h->small_sns.size();
        if (s1 == s0) continue;
        if (!forked) {
          const int ev = h->nevents++;
          h->plan.push_back(Launch{0, 0, 0, 0, 0, OP_RECORD, SB, ev});
          h->plan.push_back(Launch{0, 0, 0, 0, 0, OP_WAIT, SB + 1, ev});
          forked = true;
        }
        Launch L{K_SMALL, s0, (int)(s1 - s0), fsm, bsm, OP_LAUNCH, SB + 1, -1};
        L.aux = mx;
        L.aux2 = mxm;
        L.aux3 = bk < 9 ? mxk : 0;
        h->plan.push_back(L);
      }
    }
    auto dtop = [&](int J) { return top_markers && h->top_dist[J]; };
    int maxblk = 0;
    for (int x = h->level_off[l]; x < h->level_off[l + 1]; ++x) {
      if (h->is_small[h->level_sns[x]] || !(active(h->level_sns[x]) || dtop(h->level_sns[x]))) continue;
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
    // NEXT is split further: NEXT_a = the first inner block of outer block S+1 (all the cdiv of the
    // next step needs) stays on stream 0; NEXT_b = its other columns runs at high priority on
    // stream 1 ahead of REST(S), and the first in-block update of S+1 (same entries) waits for it.
    const long long level_p0 = (long long)h->ptasks.size();
    // in-block update direction for this level: left-looking (fewer read-modify-write passes) where
    // the level has many large supernodes (bandwidth-bound, chains overlap), right-looking where a
    // few large supernodes make the cdiv chain critical
    bool left_inner = !h->right_inner;
    if (h->left_inner_min > 0) {
      int nbig = 0;
      for (int x = h->level_off[l]; x < h->level_off[l + 1]; ++x) nbig += !h->is_small[h->level_sns[x]];
      left_inner = left_inner || nbig >= h->left_inner_min;
    }
    int pending_rest_ev = -1;      // event recorded after the latest REST launch on stream 1
    int pending_nextb_ev = -1;     // event recorded after the latest NEXT_b launch
    // multi-GPU: event after the trailing-stream reads (NEXT_b, REST) of outer block column C; the
    // broadcast into C's ring slot waits for the readers of the slot's previous block, C - ring_ns
    std::vector<int> rest_ev_of_C(maxblk / std::max(1, OUTER) + 2, -1);
    // fused cdiv (panel_kernel): one launch per outer block step does POTRF, TRSM and the in-block
    // updates of the whole outer block; NEXT is then one critical-stream launch (no NEXT_a / NEXT_b)
    // (levels with at most panel_max_sn large supernodes: where the chain is critical; wide levels
    // keep the batched launches, whose many CTAs per SM hide the short-K tiles' latency better)
    int nlarge = 0;
    for (int x = h->level_off[l]; x < h->level_off[l + 1]; ++x)
      nlarge += !h->is_small[h->level_sns[x]] && (active(h->level_sns[x]) || dtop(h->level_sns[x]));
    // (not in deterministic mode: the lookahead quarters accumulate by FP64 RED in arrival order)
    const bool panel = h->panel_mode && NB == NBMAX && OUTER <= 4 && nlarge <= h->panel_max_sn && !h->opt.deterministic;
    const bool split_next = !h->no_lookahead && !h->no_next_split;
    for (int s = 0; s < maxblk; ++s) {
      long long p0 = (long long)h->ptasks.size(), t0 = (long long)h->gtasks.size();
      double fp = 0, ft = 0, fl = 0, bp = 0, bt = 0, bl = 0, fn = 0, bn = 0, fr = 0, br = 0, fnb = 0, bnb = 0;
      std::vector<GTask> local, left, nxt, nxtb, rest;
      std::vector<std::vector<PanTask>> pan;   // per supernode: its outer block's tiles in order
      double fpan = 0, bpan = 0;
      int nd = 0;
      bool pan_next = false;
      double flf = 0, blf = 0;
      std::vector<std::pair<int, int>> bcast;   // (J, column block) finished at this step
      for (int x = h->level_off[l]; x < h->level_off[l + 1]; ++x) {
        const int J = h->level_sns[x];
        const bool dj = dtop(J);
        if (h->is_small[J] || !(dj || active(J))) continue;
        const SnInfo& I = h->sn[J];
        const int c0 = s * NB;
        if (c0 >= I.k) continue;
        const int slot = h->slot_base[J] + s;   // every diagonal block keeps its own inverse (solve)
        const int nb = std::min(NB, I.k - c0), c1 = c0 + nb;
        const int C0 = (c0 / W) * W, C1 = std::min(C0 + W, I.k);   // enclosing outer block
        auto own = [&](int col) { return !dj || blk_owner(h, J, col / W) == h->rank; };
        // fused cdiv for the outer block starting at column C: in chain-critical levels, once the rows
        // left (m - C) are few enough that the trailing update no longer hides the chain
        auto pan_at = [&](int C) { return panel && I.m - C <= h->panel_max_rows; };
        if (own(C0) && pan_at(C0)) {
          if (c0 == C0) {   // the whole outer block [C0, C1) as one set of panel tiles
            const int w = C1 - C0, nbk = (w + NB - 1) / NB;
            const int ntile = (I.m - C0 + TILE - 1) / TILE;
            std::vector<PanTask> v;
            // the lookahead update by the previous outer block (NEXT) is folded into the tiles
            // (not for a distributed top supernode: its NEXT runs on the next block's owner)
            const int pw = C0 > 0 && !dj ? W : 0;   // NEXT(C0 - W) folded here (see the NEXT emission below)
            // the diagonal region's NEXT in K = 64 quarters, its blocks (i, j <= i) in pair order, then
            // the blocks below
            for (int q = 0; pw > 0 && q < (pw + NB - 1) / NB; ++q)
              for (int i = 0; i < nbk; ++i)
                for (int j = 0; j <= i; ++j) v.push_back(PanTask{J, C0, w, i, j, slot, h->npanflags, pw, q});
            for (int i = 0; i < nbk; ++i)
              for (int j = 0; j <= i; ++j) v.push_back(PanTask{J, C0, w, i, j, slot, h->npanflags, pw, -1});
            for (int j = 0; j < nbk; ++j)
              for (int i = nbk; i < ntile; ++i) v.push_back(PanTask{J, C0, w, i, j, slot, h->npanflags, pw, -1});
            h->npanflags += 32 + 4 * std::max(0, ntile - nbk);
            pan.push_back(std::move(v));
            pan_next = pan_next || pw > 0;
            for (int c = C0; c < C1 && pw > 0; ++c) { fpan += 2.0 * pw * (double)(I.m - c); bpan += 16.0 * (double)(I.m - c); }
            for (int b = C0; b < C1; b += NB) {   // POTRF + TRSM + in-block update of inner block b
              const int nbb = std::min(NB, C1 - b), b1 = b + nbb;
              fpan += (double)nbb * nbb * nbb / 3.0 + (double)(I.m - b1) * nbb * nbb;
              bpan += 16.0 * nbb * nbb + 16.0 * (double)(I.m - b1) * nbb;
              for (int c = b1; c < C1; ++c) { fpan += 2.0 * nbb * (double)(I.m - c); bpan += 16.0 * (double)(I.m - c); }
            }
          }
        } else if (own(C0)) {
          h->ptasks.push_back(PTask{J, c0, nb, slot});
          fp += (double)nb * nb * nb / 3.0;
          bp += 16.0 * nb * nb;
          // row tiles start on an even row (16-byte aligned cp.async); rows < c1 are masked (s0 = c1)
          for (int r0 = c1 & ~1; r0 < I.m; r0 += TILE) h->gtasks.push_back(GTask{J, r0, c1, c0, nb, slot});
          ft += (double)(I.m - c1) * nb * nb;
          bt += 16.0 * (double)(I.m - c1) * nb;
          if (left_inner) {
            // left-looking inside the outer block: before its POTRF, block column [c0, c1) takes
            // the updates of the block columns [C0, c0) in one K = c0 - C0 pass (each column
            // block is read and written once per outer block instead of once per inner step)
            if (c0 > C0) {
              for_tiles(c0, I.m, c0, c1, [&](int r0, int s0) { left.push_back(GTask{J, r0, s0, C0, c0 - C0, c1}); });
              for (int c = c0; c < c1; ++c) { flf += 2.0 * (c0 - C0) * (double)(I.m - c); blf += 16.0 * (double)(I.m - c); }
            }
          } else {
            // right-looking inner update: columns [c1, C1) of this outer block, K = nb
            for_tiles(c1, I.m, c1, C1, [&](int r0, int s0) { local.push_back(GTask{J, r0, s0, c0, nb, C1}); });
            for (int c = c1; c < C1; ++c) { fl += 2.0 * nb * (double)(I.m - c); bl += 16.0 * (double)(I.m - c); }
          }
        }
        if (c1 == C1 && dj) bcast.push_back({J, C0 / W});
        // outer update after the last inner block of the outer block, K = C1 - C0 (a distributed
        // supernode: each rank updates the tiles of the column blocks it owns; W is a multiple of
        // TILE there, so no tile straddles two blocks)
        if (c1 == C1 && C1 < I.k) {
          const int C2 = std::min(C1 + W, I.k);
          if (own(C1) && (!pan_at(C1) || dj)) {   // (else folded into the next outer block's panel launch)
            const int Ca = split_next ? std::min(C1 + NB, C2) : C2;
            for_tiles(C1, I.m, C1, Ca, [&](int r0, int s0) { nxt.push_back(GTask{J, r0, s0, C0, C1 - C0, Ca}); });
            for (int c = C1; c < Ca; ++c) { fn += 2.0 * (C1 - C0) * (double)(I.m - c); bn += 16.0 * (double)(I.m - c); }
            for_tiles(Ca, I.m, Ca, C2, [&](int r0, int s0) { nxtb.push_back(GTask{J, r0, s0, C0, C1 - C0, C2}); });
            for (int c = Ca; c < C2; ++c) { fnb += 2.0 * (C1 - C0) * (double)(I.m - c); bnb += 16.0 * (double)(I.m - c); }
          }
          for_tiles(C2, I.m, C2, I.k, [&](int r0, int s0) { if (own(s0)) rest.push_back(GTask{J, r0, s0, C0, C1 - C0, I.k}); });
          for (int c = C2; c < I.k; ++c)
            if (own(c)) { fr += 2.0 * (C1 - C0) * (double)(I.m - c); br += 16.0 * (double)(I.m - c); }
        }
      }
      long long p1 = (long long)h->ptasks.size(), t1 = (long long)h->gtasks.size();
      if (!left.empty()) {   // left-looking in-block update of this step's block column, before its POTRF
        if (pending_nextb_ev >= 0) {   // same entries as NEXT_b
          h->plan.push_back(Launch{0, 0, 0, 0, 0, OP_WAIT, SB, pending_nextb_ev});
          pending_nextb_ev = -1;
        }
        long long f0 = (long long)h->gtasks.size();
        h->gtasks.insert(h->gtasks.end(), left.begin(), left.end());
        push(K_LOCAL, f0, (long long)h->gtasks.size(), flf, blf);
      }
      if (!pan.empty()) {   // task x of every outer block after the tasks < x of all of them (the
                            // diagonal-region pairs, then the tiles below, each in dependency order)
        const long long q0 = (long long)h->pantasks.size();
        size_t mx = 0;
        for (const auto& v : pan) mx = std::max(mx, v.size());
        for (int below = 0; below < 2; ++below)
          for (size_t i = 0; i < mx; ++i)
            for (const auto& v : pan) {
              if (i >= v.size()) continue;
              const bool isb = v[i].tile >= (v[i].w + NB - 1) / NB;
              if (isb == (below == 1)) h->pantasks.push_back(v[i]);
              if (!below && !isb) ++nd;
            }
        // the folded NEXT(S-1) touches the entries REST(S-2) updated: wait for it (REST(S-1) is disjoint)
        const int Cn = s / OUTER;
        if (pan_next && Cn >= 2 && rest_ev_of_C[Cn - 2] >= 0)
          h->plan.push_back(Launch{0, 0, 0, 0, 0, OP_WAIT, SB, rest_ev_of_C[Cn - 2]});
        Launch P{K_PANEL, q0, (int)((long long)h->pantasks.size() - q0), fpan, bpan, OP_LAUNCH, SB, -1};
        P.aux = h->npanlaunch++;   // sync3 index
        P.aux2 = nd;               // diagonal tiles first
        h->plan.push_back(P);
      }
      push(K_POTRF, p0, p1, fp, bp);
      push(K_TRSM, t0, t1, ft, bt);
      long long l0 = (long long)h->gtasks.size();
      h->gtasks.insert(h->gtasks.end(), local.begin(), local.end());
      if (!local.empty() && pending_nextb_ev >= 0) {   // in-block update after NEXT_b (same entries)
        h->plan.push_back(Launch{0, 0, 0, 0, 0, OP_WAIT, SB, pending_nextb_ev});
        pending_nextb_ev = -1;
      }
      push(K_LOCAL, l0, (long long)h->gtasks.size(), fl, bl);
      if (!bcast.empty()) {
        const int Cb = s / OUTER;
        if (Cb >= h->ring_ns && rest_ev_of_C[Cb - h->ring_ns] >= 0)
          h->plan.push_back(Launch{0, 0, 0, 0, 0, OP_WAIT, SB, rest_ev_of_C[Cb - h->ring_ns]});
      }
      for (const auto& jc : bcast) {   // finished block columns to the rest of their group (stream SB)
        Launch M{0, 0, 0, 0, 0, OP_BCAST, SB, -1};
        M.aux = jc.first;
        M.aux2 = jc.second;
        h->plan.push_back(M);
      }
      if (!rest.empty() && h->no_lookahead) {   // diagnostics: NEXT and REST as one launch, serial
        nxt.insert(nxt.end(), rest.begin(), rest.end());
        fn += fr; bn += br;
        rest.clear();
      }
      if (!rest.empty() || !nxtb.empty()) {   // fork NEXT_b(S), REST(S) onto stream 1 after the cdiv of block S
        const int ev = h->nevents++;
        h->plan.push_back(Launch{0, 0, 0, 0, 0, OP_RECORD, SB, ev});
        h->plan.push_back(Launch{0, 0, 0, 0, 0, OP_WAIT, SB + 1, ev});
        if (!nxtb.empty()) {
          long long b0 = (long long)h->gtasks.size();
          h->gtasks.insert(h->gtasks.end(), nxtb.begin(), nxtb.end());
          Launch NB_{K_LOCAL, b0, (int)nxtb.size(), fnb, bnb, OP_LAUNCH, SB + 1, -1};
          NB_.aux = 1;   // high priority although on the trailing stream
          h->plan.push_back(NB_);
          pending_nextb_ev = h->nevents++;
          h->plan.push_back(Launch{0, 0, 0, 0, 0, OP_RECORD, SB + 1, pending_nextb_ev});
        }
        long long r0g = (long long)h->gtasks.size();
        h->gtasks.insert(h->gtasks.end(), rest.begin(), rest.end());
        if ((long long)h->gtasks.size() > r0g)
          h->plan.push_back(Launch{K_LOCAL, r0g, (int)((long long)h->gtasks.size() - r0g), fr, br, OP_LAUNCH, SB + 1, -1});
      }
      if (!nxt.empty()) {
        if (pending_rest_ev >= 0) h->plan.push_back(Launch{0, 0, 0, 0, 0, OP_WAIT, SB, pending_rest_ev});
        long long n0 = (long long)h->gtasks.size();
        h->gtasks.insert(h->gtasks.end(), nxt.begin(), nxt.end());
        push(K_LOCAL, n0, (long long)h->gtasks.size(), fn, bn);
      }
      if (!rest.empty() || !nxtb.empty()) {
        pending_rest_ev = h->nevents++;
        h->plan.push_back(Launch{0, 0, 0, 0, 0, OP_RECORD, SB + 1, pending_rest_ev});
        rest_ev_of_C[s / OUTER] = pending_rest_ev;
      }
    }
    (void)pending_nextb_ev;
    bool s1_used = false;
    for (size_t q = plan_before; q < h->plan.size(); ++q) s1_used |= h->plan[q].stream == SB + 1;
    if (s1_used) {  // join stream 1 (small-supernode launch and trailing updates) before the level's scatter
      const int ev = h->nevents++;
      h->plan.push_back(Launch{0, 0, 0, 0, 0, OP_RECORD, SB + 1, ev});
      h->plan.push_back(Launch{0, 0, 0, 0, 0, OP_WAIT, SB, ev});
    }
    (void)pending_rest_ev;
    if (h->opt.update_mode == 1) {
      // RLB: per supernode, every block pair (B above-or-equal B') updates L_{B',B} of
      // B's ancestor directly; tiles = aligned 64-row windows intersected with the block pair
      long long r0t = (long long)h->rtasks.size();
      double fr2 = 0, br2 = 0;
      for (int x = h->level_off[l]; x < h->level_off[l + 1]; ++x) {
        const int J = h->level_sns[x];
        if (h->is_small[J] || !active(J)) continue;
        const SnInfo& I = h->sn[J];
        const int t = I.m - I.k;
        if (t <= 0) continue;
        const int base = I.k & ~1;
        const int* rJ = S.rows.data() + S.rows_ptr[J];
        for (long long b = S.blk_ptr[J]; b < S.blk_ptr[J + 1]; ++b) {
          const int P = S.blk_anc[b], qB = S.blk_q[b], nB = S.blk_len[b];
          const SnInfo& IP = h->sn[P];
          long long pr = S.rel_ptr[J];     // the (J, P) relind pair
          while (S.rel_anc[pr] != P) ++pr;
          const long long colP = rJ[qB] - S.sfirst[P];
          for (long long b2 = b; b2 < S.blk_ptr[J + 1]; ++b2) {
            const int qB2 = S.blk_q[b2], nB2 = S.blk_len[b2];
            const int posP = IP.m - 1 - S.relind[S.rel_off[pr] + (qB2 - S.rel_q0[pr])];
            const int wr0 = base + ((qB2 - base) / TILE) * TILE, wc0 = base + ((qB - base) / TILE) * TILE;
            for (int Ra = wr0; Ra < qB2 + nB2; Ra += TILE)
              for (int Rb = wc0; Rb < qB + nB; Rb += TILE) {
                const int i0 = std::max(qB2, Ra) - Ra, i1 = std::min(qB2 + nB2, Ra + TILE) - Ra;
                const int j0 = std::max(qB, Rb) - Rb, j1 = std::min(qB + nB, Rb + TILE) - Rb;
                const bool diag = b2 == b;
                if (diag && Ra + i1 - 1 < Rb + j0) continue;      // entirely above the diagonal
                RTask T{J, Ra, Rb, i0, i1, j0, j1, diag ? 1 : 0,
                        IP.off + (colP + (Rb + j0 - qB)) * IP.ld + posP + (Ra + i0 - qB2), IP.ld, 0};
                h->rtasks.push_back(T);
              }
          }
        }
        fr2 += (double)I.k * t * (t + 1);
        br2 += 8.0 * (double)t * I.k + 16.0 * 0.5 * t * (t + 1.0);
      }
      if ((long long)h->rtasks.size() > r0t)
        h->plan.push_back(Launch{K_RLB, r0t, (int)((long long)h->rtasks.size() - r0t), fr2, br2, OP_LAUNCH, SB, -1});
      h->plan_level.resize(h->plan.size(), l);
      continue;
    }
    std::vector<int> bg, bcol, bks;
    for (int x = h->level_off[l]; x < h->level_off[l + 1]; ++x) {
      const int J = h->level_sns[x];
      if (dtop(J)) {
        if (in_group(h, J, h->rank) && h->sn[J].m > h->sn[J].k) bks.push_back(J);
        continue;
      }
      if (!h->is_small[J] && active(J) && h->sn[J].m > h->sn[J].k) bg.push_back(J);
    }
    const int nbc = h->opt.deterministic ? colour_supernodes(h, bg, bcol) : 1;
    if (!h->opt.deterministic) bcol.assign(bg.size(), 0);
    for (int col = 0; col < nbc; ++col) {   // one launch per colour class (one class unless deterministic)
      long long s0g = (long long)h->gtasks.size();
      double fs = 0, bs = 0;
      for (size_t x = 0; x < bg.size(); ++x) {
        if (bcol[x] != col) continue;
        const int J = bg[x];
        const SnInfo& I = h->sn[J];
        const int t = I.m - I.k;
        const int base = I.k & ~1;
        for_tiles(base, I.m, base, I.m, [&](int r0, int c0) { h->gtasks.push_back(GTask{J, r0, c0, 0, 0, 0}); });
        fs += (double)I.k * t * (t + 1);
        bs += 8.0 * (double)t * I.k + 16.0 * 0.5 * t * (t + 1.0);
      }
      push(K_SCATTER, s0g, (long long)h->gtasks.size(), fs, bs);
      if (h->opt.deterministic && !h->plan.empty() && h->plan.back().kind == K_SCATTER && h->plan.back().off == s0g)
        h->plan.back().aux = 1;
    }
    if (!bks.empty()) {
      // distributed top supernodes: this rank's partial U_J over the block columns it owns (C = cr,
      // cr + g, ...: cyclic ownership), RED into its update block of J (dist_redirect)
      const int W = h->outer * h->nb;
      long long s0g = (long long)h->gtasks.size();
      double fs = 0, bs = 0;
      for (int J : bks) {
        const SnInfo& I = h->sn[J];
        const int g = h->grp_hi[J] - h->grp_lo[J], nblk = (I.k + W - 1) / W;
        const int cr = ((h->rank - h->top_owner[J]) % g + g) % g;
        if (cr >= nblk) continue;
        const int cnt = (nblk - 1 - cr) / g + 1;
        double cols = 0;
        for (int i = 0; i < cnt; ++i) cols += std::min(W, I.k - (cr + i * g) * W);
        const int base = I.k & ~1;
        const double t = I.m - I.k;
        for_tiles(base, I.m, base, I.m, [&](int r0, int c0) { h->gtasks.push_back(GTask{J, r0, c0, cr * W, cnt, g * W}); });
        fs += cols * t * (t + 1);
        bs += 8.0 * t * cols + 16.0 * 0.5 * t * (t + 1.0);
      }
      push(K_SCATTER, s0g, (long long)h->gtasks.size(), fs, bs);
      if (!h->plan.empty() && h->plan.back().kind == K_SCATTER && h->plan.back().off == s0g) h->plan.back().aux = 2;
    }
    if (top_markers && l + 1 < h->nexch && !h->exch_runs[l + 1].empty()) {
      // the level's partial U_J go to the owners of their destination block columns
      Launch M{0, 0, 0, 0, 0, OP_EXCHANGE, SB, -1};
      M.aux = l + 1;
      h->plan.push_back(M);
    }
    h->plan_level.resize(h->plan.size(), l);
  }
  if (record_solve) h->small_level_off.push_back((int)h->small_sns.size());
}


// Level solve tasks (sync-free blocked triangular solve, see solve_fwd_level_kernel).  Order inside
// a level = the ticket order: forward, triangle blocks b = 0, 1, ... interleaved over the level's
// supernodes, then the rows below the triangles; backward, the chunks below the triangles, then the
// triangle column blocks from the last to the first.  A task only waits for tasks before it.
template <class Active>
static void build_solve_tasks(spchol_handle* h, Active active, bool append = false) {
  const Symbolic& S = h->S;
  const int NB = h->nb;
  if (!append) {
    h->stasks.clear();
    h->ssolve.clear();
  }
  h->sfwd_off.assign(S.nlevels + 1, 0);
  h->sbwd_off.assign(S.nlevels + 1, 0);
  for (int l = 0; l < S.nlevels; ++l) {
    std::vector<int> big;
    int maxblk = 0;
    for (int x = h->level_off[l]; x < h->level_off[l + 1]; ++x) {
      const int J = h->level_sns[x];
      if (h->is_small[J] || h->sn[J].k == 0 || !active(J)) continue;
      big.push_back(J);
      maxblk = std::max(maxblk, (h->sn[J].k + NB - 1) / NB);
    }
    h->sfwd_off[l] = (long long)h->stasks.size();
    for (int b = 0; b < maxblk; ++b)
      for (int J : big) {
        const SnInfo& I = h->sn[J];
        if (b * NB >= I.k) continue;
        const int nb = std::min(NB, I.k - b * NB);
        h->stasks.push_back(STask{J, 0, b, nb, b * NB, b * NB + nb, h->slot_base[J] + b, 0, 0, (I.k + NB - 1) / NB});
      }
    for (int J : big) {
      const SnInfo& I = h->sn[J];
      for (int q0 = I.k; q0 < I.m; q0 += 64)
        h->stasks.push_back(STask{J, 1, 0, 0, q0, std::min(q0 + 64, I.m), h->slot_base[J], 0, 0, (I.k + NB - 1) / NB});
    }
    h->sbwd_off[l] = (long long)h->stasks.size();
    for (int J : big) {
      const SnInfo& I = h->sn[J];
      const int nblk = (I.k + NB - 1) / NB;
      for (int b = 0; b < nblk; ++b)
        for (int q0 = I.k; q0 < I.m; q0 += SOLVE_RCHUNK)
          h->stasks.push_back(STask{J, 2, b, std::min(NB, I.k - b * NB), q0, std::min(q0 + SOLVE_RCHUNK, I.m), h->slot_base[J] + b, 0, 0, nblk});
    }
    for (int d = 0; d < maxblk; ++d)
      for (int J : big) {
        const SnInfo& I = h->sn[J];
        const int nblk = (I.k + NB - 1) / NB, b = nblk - 1 - d;
        if (b < 0) continue;
        const int need = (I.m - I.k + SOLVE_RCHUNK - 1) / SOLVE_RCHUNK;
        h->stasks.push_back(STask{J, 3, b, std::min(NB, I.k - b * NB), b * NB, b * NB + std::min(NB, I.k - b * NB), h->slot_base[J] + b, need, 0, nblk});
      }
  }
  h->sfwd_off[S.nlevels] = h->sbwd_off[S.nlevels] = (long long)h->stasks.size();
  h->nticket = 2 * (size_t)S.nlevels;
  h->ssolve_off.assign(3 * S.nlevels + 1, 0);
  for (int l = 0; l < S.nlevels; ++l)
    for (int cl = 0; cl < 3; ++cl) {
      h->ssolve_off[3 * l + cl] = (int)h->ssolve.size();
      for (int x = h->level_off[l]; x < h->level_off[l + 1]; ++x) {
        const int J = h->level_sns[x];
        const SnInfo& I = h->sn[J];
        if (!h->is_small[J] || (I.m > 64) + (I.m > 128) != cl || !active(J)) continue;
        h->ssolve.push_back(SmallSolve{I.off, S.rows_ptr[J], I.ld, I.m, I.k, S.sfirst[J]});
      }
    }
  h->ssolve_off[3 * S.nlevels] = (int)h->ssolve.size();
}

// Memory-capped mode (f-4; "RLB-v2" caps GPU memory, P:568 RL runs out of it): the tree is
// split into a resident top and subtree batches that share one device window.  A subtree whose panels
// fit the window W is a unit; units are packed in postorder into batches of at most W; every supernode
// above them stays resident.  W is the largest window with W + top(W) + fixed costs <= the cap (the
// top shrinks as W grows).  Returns false if no window fits.
static bool capped_layout(spchol_handle* h) {
  const Symbolic& S = h->S;
  const int ns = S.nsuper, NB = h->nb;
  auto al = [](long long x) { return (x + 255) / 256 * 256; };   // 2 KB-aligned regions
  std::vector<long long> pb(ns), sb(ns, 0);
  for (int J = 0; J < ns; ++J) pb[J] = al((long long)h->sn[J].ld * h->sn[J].k);
  for (int J = 0; J < ns; ++J) {
    sb[J] += pb[J];
    if (S.sparent[J] >= 0) sb[S.sparent[J]] += sb[J];
  }
  // inverse slots as usual (all resident)
  h->slot_base.assign(ns, 0);
  int slot = 0;
  for (int J = 0; J < ns; ++J) {
    if (h->is_small[J]) continue;
    h->slot_base[J] = slot;
    slot += (h->sn[J].k + NB - 1) / NB;
  }
  h->nslots_total = slot;
  // the cap bounds the factor's device storage: the panel window + the resident top panels + the kept
  // diagonal-block inverses (SPCHOL_Q_ARENA_BYTES); metadata comes on top (SPCHOL_Q_DEVICE_BYTES)
  const double fixed = 8.0 * NBMAX * NBMAX * slot;
  const double budget = (double)h->opt.device_mem_cap - fixed;
  std::vector<long long> cand(sb.begin(), sb.end());
  std::sort(cand.begin(), cand.end());
  cand.erase(std::unique(cand.begin(), cand.end()), cand.end());
  long long W = -1;
  for (size_t i = cand.size(); i-- > 0;) {
    long long top = 0;
    for (int J = 0; J < ns; ++J) if (sb[J] > cand[i]) top += pb[J];
    if ((double)(cand[i] + top) * 8.0 <= budget) { W = cand[i]; break; }
  }
  if (W < 0) return false;
  // units = maximal subtrees with sb <= W (contiguous in postorder), packed into batches
  h->batch.assign(ns, -1);
  std::vector<long long> blen;
  long long cur = -1;
  int J = 0;
  while (J < ns) {
    // the unit root is the highest ancestor of J whose subtree still fits
    int root = J;
    if (sb[J] > W) { ++J; continue; }      // a top supernode
    while (S.sparent[root] >= 0 && sb[S.sparent[root]] <= W) root = S.sparent[root];
    if (cur < 0 || blen.back() + sb[root] > W) { blen.push_back(0); cur = (long long)blen.size() - 1; }
    for (int q = J; q <= root; ++q) h->batch[q] = (int)cur;   // J .. root = root's subtree (postorder)
    blen.back() += sb[root];
    J = root + 1;
  }
  h->nbatch = (int)blen.size();
  // offsets: each batch from 0 inside the window; the top after the window; host copy per batch
  h->batch_len.assign(h->nbatch, 0);
  h->batch_host.assign(h->nbatch + 1, 0);
  h->host_off.assign(ns, -1);
  long long wmax = 0;
  for (int b = 0; b < h->nbatch; ++b) wmax = std::max(wmax, blen[b]);
  h->window_doubles = al(wmax);
  h->top_base = h->window_doubles;
  long long toff = h->top_base;
  for (int q = 0; q < ns; ++q) {
    const int b = h->batch[q];
    if (b < 0) {
      h->sn[q].off = toff;
      toff += pb[q];
    } else {
      h->sn[q].off = h->batch_len[b];
      h->host_off[q] = h->batch_len[b];   // relative to the batch's host base (fixed below)
      h->batch_len[b] += pb[q];
    }
  }
  for (int b = 0; b < h->nbatch; ++b) h->batch_host[b + 1] = h->batch_host[b] + h->batch_len[b];
  for (int q = 0; q < ns; ++q) if (h->batch[q] >= 0) h->host_off[q] += h->batch_host[h->batch[q]];
  h->panel_doubles = toff;
  h->capped = true;
  return true;
}

static void build_plan(spchol_handle* h) {
  const Symbolic& S = h->S;
  const int ns = S.nsuper, NB = h->nb;
  h->sn.resize(ns);
  h->panel_off.assign(ns + 1, 0);
  h->work.assign(ns, 0.0);
  std::vector<double>& work = h->work;
  for (int J = 0; J < ns; ++J) {
    int k = S.sfirst[J + 1] - S.sfirst[J];
    int m = (int)(S.rows_ptr[J + 1] - S.rows_ptr[J]);
    int ld = m + (m & 1);
    h->sn[J].ld = ld; h->sn[J].m = m; h->sn[J].k = k; h->sn[J].ucol = -1;
    for (int c = 0; c < k; ++c) work[J] += (double)(m - c) * (double)(m - c);
    h->flops_exec += work[J];
    h->update_entries += 0.5 * (double)(m - k) * (double)(m - k + 1);
  }
  // subtree-to-GPU mapping (multi-GPU): owner[J] = rank, or -1 for the top (separator) supernodes
  {
    std::vector<int> lo, hi;
    proportional_map(S, work, h->world, h->owner, &lo, &hi);
    assign_top_owners(work, h->owner, lo, hi, S.level, h->world, h->top_owner);
    h->grp_lo = lo;
    h->grp_hi = hi;
    h->top_by_level.assign(S.nlevels, {});
    if (h->world > 1)
      for (int J = 0; J < ns; ++J) if (h->owner[J] < 0) h->top_by_level[S.level[J]].push_back(J);
  }
  // levels
  h->level_off.assign(S.nlevels + 1, 0);
  for (int J = 0; J < ns; ++J) h->level_off[S.level[J] + 1]++;
  for (int l = 0; l < S.nlevels; ++l) h->level_off[l + 1] += h->level_off[l];
  h->level_sns.assign(ns, 0);
  {
    std::vector<int> nx(h->level_off.begin(), h->level_off.end() - 1);
    for (int J = 0; J < ns; ++J) h->level_sns[nx[S.level[J]]++] = J;
  }
  // fused small-supernode path: k <= small_max_k, m <= 256, m k <= SMALL_MAXELEMS (shared memory);
  // multi-GPU top supernodes always take the blocked path (their solve steps use the kept inverses)
  const int kmax = h->opt.small_max_k < 0 ? 0 : (h->opt.small_max_k == 0 ? SMALL_MAXK : std::min(h->opt.small_max_k, SMALL_MAXK));
  h->is_small.assign(ns, 0);
  for (int J = 0; J < ns; ++J) {
    const SnInfo& I = h->sn[J];
    h->is_small[J] = I.k <= kmax && I.m <= SMALL_MAXM && (long long)I.m * I.k <= SMALL_MAXELEMS &&
                     !(h->world > 1 && h->owner[J] < 0);
  }
  // distributed top supernodes (multi-GPU): large enough that splitting the cdiv and U_J over the
  // rank group beats the block-column broadcasts it costs; the outer block width W must be a power
  // of two (block columns = whole VMM pages, K-split chunk arithmetic)
  h->top_dist.assign(ns, 0);
  const int W = h->outer * NB;
  if (h->world > 1 && W % TILE == 0 && (W & (W - 1)) == 0 && h->opt.update_mode == 0)
    for (int J = 0; J < ns; ++J)
      h->top_dist[J] = h->owner[J] < 0 && h->grp_hi[J] - h->grp_lo[J] > 1 && !h->is_small[J] && work[J] >= h->dist_min_flops;
  bool capped_fail = false;
  if (h->world == 1 && h->opt.device_mem_cap > 0) {
    capped_fail = !capped_layout(h);
  } else if (h->world == 1) {
    // panel arena: supernodes in order
    long long off = 0;
    for (int J = 0; J < ns; ++J) {
      h->sn[J].off = off;
      off += (long long)h->sn[J].ld * h->sn[J].k;
    }
    h->panel_doubles = off;
    // persistent diagonal-block inverse slots (factor TRSM + solve)
    h->slot_base.assign(ns, 0);
    int slot = 0;
    for (int J = 0; J < ns; ++J) {
      if (h->is_small[J]) continue;
      h->slot_base[J] = slot;
      slot += (h->sn[J].k + NB - 1) / NB;
    }
    h->nslots_total = slot;
  } else {
    dist_layout(h);   // per-rank arena: own subtrees, owned top block columns, ring aliases
  }
  for (int J = 0; J < ns; ++J) h->panel_off[J] = h->sn[J].off;
  h->panel_off[ns] = h->panel_doubles;
  if (h->capped) {   // exported layout: the batches' host copy, then the resident top (distinct offsets)
    const long long hb = h->batch_host[h->nbatch];
    for (int J = 0; J < ns; ++J) h->panel_off[J] = h->batch[J] >= 0 ? h->host_off[J] : hb + h->sn[J].off - h->top_base;
    h->panel_off[ns] = hb + h->panel_doubles - h->top_base;
  }
  if (capped_fail) { h->capped = false; h->nbatch = -1; return; }
  if (h->capped) {
    // batch by batch (each in the window), then the resident top; the solve per segment
    h->plan_batch.assign(h->nbatch + 1, 0);
    h->segs.clear();
    for (int b = 0; b < h->nbatch; ++b) {
      h->plan_batch[b] = h->plan.size();
      append_levels(h, [h, b](int J) { return h->batch[J] == b; }, false);
      build_solve_tasks(h, [h, b](int J) { return h->batch[J] == b; }, b > 0);
      h->segs.push_back({h->sfwd_off, h->sbwd_off, h->ssolve_off});
    }
    h->plan_batch[h->nbatch] = h->plan.size();
    append_levels(h, [h](int J) { return h->batch[J] < 0; }, false);
    build_solve_tasks(h, [h](int J) { return h->batch[J] < 0; }, h->nbatch > 0);
    h->segs.push_back({h->sfwd_off, h->sbwd_off, h->ssolve_off});
    h->nticket = 2 * (size_t)S.nlevels * h->segs.size();
    h->plan_factor_begin = 0;
    h->plan_all_end = h->plan_a_end = h->plan.size();
    return;
  }
  if (h->world == 1) {
    // the whole tree (the solve's structure; the single-GPU factor when nvr == 1)
    append_levels(h, [](int) { return true; }, true);
    build_solve_tasks(h, [](int) { return true; });
    h->plan_all_end = h->plan.size();
    h->plan_factor_begin = 0;
    if (h->nvr > 1) {
      // single GPU, subtree concurrency: proportional map onto nvr virtual ranks; each virtual rank's
      // subtrees run on their own (critical, trailing) stream pair, the top supernodes after all of
      // them have joined stream 0
      std::vector<int> vown;
      proportional_map(S, work, h->nvr, vown);
      h->plan_factor_begin = h->plan.size();
      for (int v = 0; v < h->nvr; ++v) append_levels(h, [&vown, v](int J) { return vown[J] == v; }, false, 2 * v);
      for (int v = 1; v < h->nvr; ++v) {
        const int ev = h->nevents++;
        h->plan.push_back(Launch{0, 0, 0, 0, 0, OP_RECORD, 2 * v, ev});
        h->plan.push_back(Launch{0, 0, 0, 0, 0, OP_WAIT, 0, ev});
      }
      append_levels(h, [&vown](int J) { return vown[J] < 0; }, false, 0);
      h->plan_all_end = h->plan.size();
    }
    h->plan_a_end = h->plan.size();
    return;
  }
  // multi-GPU: phase A (own subtrees), the boundary-block exchange, phase C (top levels)
  dist_exchange_plan(h);
  const int me = h->rank;
  h->plan_all_end = h->plan_factor_begin = 0;
  append_levels(h, [h, me](int J) { return h->owner[J] == me; }, false);
  h->plan_a_end = h->plan.size();
  if (!h->exch_runs[0].empty()) {
    Launch M{0, 0, 0, 0, 0, OP_EXCHANGE, 0, -1};
    M.aux = 0;
    h->plan.push_back(M);
    h->plan_level.resize(h->plan.size(), -1);
  }
  append_levels(h, [h, me](int J) { return h->owner[J] < 0 && h->top_owner[J] == me; }, false, 0, true);
  for (size_t i = h->plan_a_end; i < h->plan.size(); ++i)
    if (h->plan[i].op == OP_EXCHANGE || h->plan[i].op == OP_BCAST) h->markers.push_back(i);
  build_solve_tasks(h, [h, me](int J) { return h->owner[J] == me; });
  dist_solve_plan(h);
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
  if (h->world > 1) dist_redirect(h, posmap, ucb);   // updates leaving the rank go to its update blocks
  std::vector<long long> amap(h->capped ? 0 : S.nnzA);
  if (h->capped) {
    // memory-capped: A's entries grouped by batch (the window's current occupant), the top's last
    h->ainit_off.assign(h->nbatch + 2, 0);
    for (long long e = 0; e < S.nnzA; ++e) {
      const int b = h->batch[S.snode[S.a_col[e]]];
      h->ainit_off[(b < 0 ? h->nbatch : b) + 1]++;
    }
    for (int b = 0; b <= h->nbatch; ++b) h->ainit_off[b + 1] += h->ainit_off[b];
    h->ainit_idx.assign(S.nnzA, 0);
    h->ainit_dst.assign(S.nnzA, 0);
    std::vector<long long> nx(h->ainit_off.begin(), h->ainit_off.end() - 1);
    for (long long e = 0; e < S.nnzA; ++e) {
      const int c = S.a_col[e], J = S.snode[c], b = h->batch[J];
      const long long x = nx[b < 0 ? h->nbatch : b]++;
      h->ainit_idx[x] = e;
      h->ainit_dst[x] = h->sn[J].off + (long long)(c - S.sfirst[J]) * h->sn[J].ld + S.a_pos[e];
    }
  }
  for (long long e = 0; e < (long long)amap.size(); ++e) {
    const int c = S.a_col[e], J = S.snode[c];
    amap[e] = h->sn[J].off + (long long)(c - S.sfirst[J]) * h->sn[J].ld + S.a_pos[e];
    // multi-GPU: a rank initialises the entries of the columns it holds
    if (h->world > 1 && !dist_amap_mine(h, c)) amap[e] = -1;
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
    int nstreams = 2;
    for (const Launch& L : h->plan) nstreams = std::max(nstreams, L.stream + 1);
    h->pstreams.assign(nstreams, nullptr);
    h->join_events.assign(nstreams, nullptr);
    for (int i = 0; i < nstreams; ++i) {
      CK(cudaStreamCreateWithPriority(&h->pstreams[i], cudaStreamNonBlocking, (i & 1) ? lo : hi));
      CK(cudaEventCreateWithFlags(&h->join_events[i], cudaEventDisableTiming));
    }
    CK(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
    if (h->world == 1 && !h->capped) {
      CK(cudaStreamCreateWithFlags(&h->zstream, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&h->ev_zs, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&h->ev_zd, cudaEventDisableTiming));
    }
  }
  h->plan_events.resize(h->nevents);
  for (auto& e : h->plan_events) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  g_dev_bytes = 0;
  if (h->world > 1) {
    int rc = dist_setup_device(h);   // per-rank arena (VMM), inverse slots, exchange metadata
    if (rc) return rc;
  } else {
    CK(dalloc(&h->d_panels, (size_t)h->panel_doubles));
  }
  CK(dalloc(&h->d_avals, (size_t)S.nnzA));
  CK(upload(&h->d_amap, amap));
  if (h->capped) {
    CK(upload(&h->d_ainit_idx, h->ainit_idx));
    CK(upload(&h->d_ainit_dst, h->ainit_dst));
    CK(cudaMallocHost((void**)&h->h_panels, sizeof(double) * (size_t)std::max(1LL, h->batch_host[h->nbatch])));
  }
  CK(upload(&h->d_ucol_base, ucb));
  CK(upload(&h->d_ucol_map, ucm));
  CK(upload(&h->d_posmap, posmap));
  CK(upload(&h->d_sn, h->sn));
  CK(upload(&h->d_sfirst, S.sfirst));
  CK(upload(&h->d_gtasks, h->gtasks));
  CK(upload(&h->d_rtasks, h->rtasks));
  CK(upload(&h->d_ptasks, h->ptasks));
  CK(upload(&h->d_pantasks, h->pantasks));
  CK(dalloc(&h->d_pansync, (size_t)h->npanflags + 3 * (size_t)h->npanlaunch));
  if (h->world == 1) CK(dalloc(&h->d_linv, (size_t)std::max(1, h->nslots_total) * NBMAX * NBMAX));
  if (h->use_tma) {
    // TMA descriptors: panel J as a 2D tensor (m_J rows contiguous, k_J columns, row stride ld_J),
    // boxes of 16 rows x 8 columns with 128-byte swizzle; rows >= m_J / columns >= k_J read as 0
    PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q));
    if (!encode || q != cudaDriverEntryPointSuccess) return fail(SPCHOL_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    std::vector<CUtensorMap> maps(std::max(1, ns));
    std::memset(maps.data(), 0, maps.size() * sizeof(CUtensorMap));
    const cuuint32_t box[2] = {(cuuint32_t)TMA_BOX_ROWS, (cuuint32_t)TMA_BOX_COLS}, es[2] = {1, 1};
    for (int J = 0; J < ns; ++J) {
      const SnInfo& I = h->sn[J];
      if (h->is_small[J] || I.k == 0) continue;
      const cuuint64_t dims[2] = {(cuuint64_t)I.m, (cuuint64_t)I.k};
      const cuuint64_t strides[1] = {(cuuint64_t)I.ld * sizeof(double)};
      CUresult r = encode(&maps[J], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, h->d_panels + I.off, dims, strides, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) return fail(SPCHOL_ERR_CUDA, "cuTensorMapEncodeTiled(panel) failed: " + std::to_string((int)r));
    }
    CK(cudaMalloc(&h->d_tmaps, maps.size() * sizeof(CUtensorMap)));
    CK(cudaMemcpy(h->d_tmaps, maps.data(), maps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice));
    CUtensorMap lm;
    std::memset(&lm, 0, sizeof(lm));
    const cuuint64_t ldims[2] = {(cuuint64_t)NBMAX, (cuuint64_t)std::max(1, h->nslots_total) * NBMAX};
    const cuuint64_t lstr[1] = {(cuuint64_t)NBMAX * sizeof(double)};
    CUresult r = encode(&lm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, h->d_linv, ldims, lstr, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(SPCHOL_ERR_CUDA, "cuTensorMapEncodeTiled(linv) failed: " + std::to_string((int)r));
    CK(cudaMalloc(&h->d_tmap_linv, sizeof(CUtensorMap)));
    CK(cudaMemcpy(h->d_tmap_linv, &lm, sizeof(lm), cudaMemcpyHostToDevice));
  }
  CK(dalloc(&h->d_fail, 1));
  CK(upload(&h->d_rows_ptr, std::vector<long long>(S.rows_ptr.begin(), S.rows_ptr.end())));
  CK(upload(&h->d_rows, S.rows));
  CK(upload(&h->d_perm, S.perm_final));
  CK(upload(&h->d_level_sns, h->level_sns));
  CK(upload(&h->d_small_sns, h->small_sns));
  CK(upload(&h->d_stasks, h->stasks));
  CK(upload(&h->d_ssolve, h->ssolve));
  CK(dalloc(&h->d_sflags, (size_t)3 * std::max(1, h->nslots_total) + h->nticket + 1));
  CK(dalloc(&h->d_y, (size_t)S.n * SOLVE_NRMAX));
  CK(dalloc(&h->d_y2, (size_t)S.n * SOLVE_NRMAX));
  h->device_bytes = g_dev_bytes;
  return SPCHOL_OK;
}

static void free_device(spchol_handle* h) {
  for (void* c : h->grp_comms) if (c && g_nccl.destroy) g_nccl.destroy(c);
  if (h->nccl_comm && g_nccl.destroy) g_nccl.destroy(h->nccl_comm);
  for (int i = 0; i < 3; ++i) {
    if (h->solve_gexec[i]) cudaGraphExecDestroy(h->solve_gexec[i]);
    if (h->solve_graph[i]) cudaGraphDestroy(h->solve_graph[i]);
  }
  if (h->gexec) cudaGraphExecDestroy(h->gexec);
  if (h->graph) cudaGraphDestroy(h->graph);
  if (h->gexec_nz) cudaGraphExecDestroy(h->gexec_nz);
  if (h->graph_nz) cudaGraphDestroy(h->graph_nz);
  if (h->zstream) cudaStreamDestroy(h->zstream);
  if (h->ev_zs) cudaEventDestroy(h->ev_zs);
  if (h->ev_zd) cudaEventDestroy(h->ev_zd);
  if (h->world > 1) dist_free_device(h);   // the VMM arenas (d_panels, d_linv)
  if (h->h_panels) cudaFreeHost(h->h_panels);
  h->h_panels = nullptr;
  if (h->d_ainit_idx) cudaFree(h->d_ainit_idx);
  if (h->d_ainit_dst) cudaFree(h->d_ainit_dst);
  void* ptrs[] = {h->d_ssolve, h->d_stasks, h->d_sflags, h->d_rtasks, h->d_tmaps, h->d_tmap_linv, h->d_small_sns, h->d_diag_idx, h->d_panels, h->d_avals, h->d_linv, h->d_y, h->d_y2, h->d_amap, h->d_ucol_base, h->d_ucol_map,
                  h->d_rows_ptr, h->d_posmap, h->d_sfirst, h->d_rows, h->d_perm, h->d_level_sns, h->d_sn,
                  h->d_gtasks, h->d_ptasks, h->d_pantasks, h->d_pansync, h->d_fail};
  for (void* p : ptrs) if (p) cudaFree(p);
  for (cudaEvent_t e : h->ev_pool) cudaEventDestroy(e);
  for (cudaEvent_t e : h->plan_events) if (e) cudaEventDestroy(e);
  for (cudaStream_t x : h->pstreams) if (x) cudaStreamDestroy(x);
  for (cudaEvent_t e : h->join_events) if (e) cudaEventDestroy(e);
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  if (h->ev_join) cudaEventDestroy(h->ev_join);
  if (h->own_stream) cudaStreamDestroy(h->own_stream);
}

extern "C" int spchol_set_values(spchol_handle* h, const double* values);

// Everything after the symbolic phase: validation of the options, launch plan, device state.
static int finish_handle(spchol_handle* h) {
  if (h->opt.block) {
    if (h->opt.block < 8 || h->opt.block > NBMAX || h->opt.block % 8) return fail(SPCHOL_ERR_VALIDATION, "block must be a multiple of 8 in [8, 64]");
    h->nb = h->opt.block;
  }
  if (h->opt.update_mode < 0 || h->opt.update_mode > 1) return fail(SPCHOL_ERR_VALIDATION, "update_mode must be 0 (RL) or 1 (RLB)");
  if (h->opt.dist_world < 1 || h->opt.dist_rank < 0 || h->opt.dist_rank >= h->opt.dist_world)
    return fail(SPCHOL_ERR_VALIDATION, "need 0 <= dist_rank < dist_world");
  h->rank = h->opt.dist_rank;
  h->world = h->opt.dist_world;
  h->nvr = h->opt.subtree_streams == 0 ? 4 : std::max(1, std::min(16, (int)h->opt.subtree_streams));
  if (h->opt.deterministic) {
    if (h->opt.update_mode != 0) return fail(SPCHOL_ERR_VALIDATION, "deterministic requires update_mode 0 (RL)");
    h->nvr = 1;   // concurrent subtrees would update the shared top panels in an unordered way
  }
  if (h->world > 1 && (h->opt.update_mode != 0 || h->opt.deterministic))
    return fail(SPCHOL_ERR_VALIDATION, "multi-GPU (dist_world > 1) supports update_mode 0 without deterministic");
  if (const char* e = getenv("SPCHOL_NO_LOOKAHEAD")) h->no_lookahead = atoi(e) != 0;
  if (const char* e = getenv("SPCHOL_NO_NEXT_SPLIT")) h->no_next_split = atoi(e) != 0;
  if (const char* e = getenv("SPCHOL_LEFT_INNER")) h->right_inner = atoi(e) == 0;
  if (const char* e = getenv("SPCHOL_LEFT_INNER_MIN")) h->left_inner_min = std::max(0, atoi(e));
  if (const char* e = getenv("SPCHOL_REST_SMEM")) h->rest_smem = std::max(0, std::min(112 * 1024, atoi(e)));
  if (const char* e = getenv("SPCHOL_MAX_LEVEL")) h->max_level = atoi(e);
  if (const char* e = getenv("SPCHOL_TMA")) h->use_tma = atoi(e) != 0 && h->world == 1;
  if (const char* e = getenv("SPCHOL_OUTER")) h->outer = std::max(1, atoi(e));
  if (const char* e = getenv("SPCHOL_DIST_MINFLOPS")) h->dist_min_flops = atof(e);
  if (const char* e = getenv("SPCHOL_RING_NS")) h->ring_ns = std::max(2, atoi(e));   // diagnostics
  if (const char* e = getenv("SPCHOL_PANEL")) h->panel_mode = atoi(e) != 0;
  if (const char* e = getenv("SPCHOL_PANEL_GRID")) h->panel_grid = std::max(0, atoi(e));
  if (const char* e = getenv("SPCHOL_PANEL_MAX_SN")) h->panel_max_sn = atoi(e);
  if (const char* e = getenv("SPCHOL_PANEL_MAX_ROWS")) h->panel_max_rows = atoi(e);
  if (const char* e = getenv("SPCHOL_SMALL_WARP")) h->small_warp = atoi(e) != 0;
  if (const char* e = getenv("SPCHOL_SMALL_WARP_MAXM")) h->small_warp_maxm = std::max(0, std::min(128, atoi(e)));
  if (h->opt.device_mem_cap < 0 || (h->opt.device_mem_cap > 0 && h->world > 1))
    return fail(SPCHOL_ERR_VALIDATION, "device_mem_cap must be >= 0 and needs dist_world == 1");
  build_plan(h);
  if (h->opt.device_mem_cap > 0 && !h->capped)
    return fail(SPCHOL_ERR_DEVICE_OOM, "device_mem_cap: the resident top of the supernodal tree alone exceeds the cap");
  if (h->opt.device < 0) return SPCHOL_OK;   // host-only analysis (no device state)
  int rc = setup_device(h);
  if (rc != SPCHOL_OK) free_device(h);
  return rc;
}

// spchol_dist_init: the process's rank / world / communicator id, applied by later analyze calls
namespace {
struct DistInit { bool set = false; int32_t rank = 0, world = 1; char uid[128]; };
DistInit g_dist_init;
std::mutex g_dist_init_mu;
}
extern "C" int spchol_dist_init(int32_t rank, int32_t world, const void* nccl_unique_id) {
  std::lock_guard<std::mutex> lock(g_dist_init_mu);
  if (world == 1) { g_dist_init.set = false; return SPCHOL_OK; }
  if (world < 1 || rank < 0 || rank >= world || !nccl_unique_id) return fail(SPCHOL_ERR_VALIDATION, "need 0 <= rank < world and an id");
  g_dist_init.set = true;
  g_dist_init.rank = rank;
  g_dist_init.world = world;
  std::memcpy(g_dist_init.uid, nccl_unique_id, 128);
  return SPCHOL_OK;
}
// apply spchol_dist_init to options left at dist_world == 1; returns whether to attach afterwards
static bool apply_dist_init(spchol_options& o, char* uid) {
  std::lock_guard<std::mutex> lock(g_dist_init_mu);
  if (!g_dist_init.set || o.dist_world != 1) return false;
  o.dist_rank = g_dist_init.rank;
  o.dist_world = g_dist_init.world;
  std::memcpy(uid, g_dist_init.uid, 128);
  return true;
}
extern "C" int spchol_dist_attach_nccl(spchol_handle* h, const void* unique_id128);

extern "C" int spchol_analyze(int64_t n, const int64_t* colptr, const int32_t* rowidx, const double* values,
                              const int32_t* perm, const spchol_options* opt, spchol_handle** out) {
  if (!out) return fail(SPCHOL_ERR_VALIDATION, "out is NULL");
  *out = nullptr;
  spchol_handle* h = new spchol_handle();
  if (opt) h->opt = *opt; else spchol_default_options(&h->opt);
  char uid[128];
  const bool attach = apply_dist_init(h->opt, uid);
  Nvtx nv("spchol_analyze");
  std::string err;
  int rc = analyze_symbolic(n, colptr, rowidx, perm, h->opt.merge_cap, h->opt.partition_refinement, h->S, err);
  if (rc != SPCHOL_OK) { delete h; return fail(rc, err); }
  rc = finish_handle(h);
  if (rc != SPCHOL_OK) { delete h; return rc; }
  if (values && h->opt.device >= 0) {
    rc = spchol_set_values(h, values);
    if (rc != SPCHOL_OK) { free_device(h); delete h; return rc; }
  }
  if (attach && h->opt.device >= 0) {
    rc = spchol_dist_attach_nccl(h, uid);
    if (rc != SPCHOL_OK) { free_device(h); delete h; return rc; }
  }
  *out = h;
  return SPCHOL_OK;
}


// ------------------------------------------------------------------------------------- serialization
// Binary file: magic, version, then every field of the symbolic analysis (scalars, then each array
// as <int64 count><raw data>).  A loaded handle rebuilds the launch plan and device state from it.
namespace {
constexpr uint64_t SPCHOL_MAGIC = 0x4C4F484350534250ull;   // "PBSPCHOL"
constexpr uint64_t SPCHOL_FORMAT = 1;
template <class T>
bool wvec(FILE* f, const std::vector<T>& v) {
  const int64_t n = (int64_t)v.size();
  return fwrite(&n, sizeof n, 1, f) == 1 && (n == 0 || fwrite(v.data(), sizeof(T), (size_t)n, f) == (size_t)n);
}
template <class T>
bool rvec(FILE* f, std::vector<T>& v) {
  int64_t n = 0;
  if (fread(&n, sizeof n, 1, f) != 1 || n < 0 || n > (int64_t)1 << 40) return false;
  v.resize((size_t)n);
  return n == 0 || fread(v.data(), sizeof(T), (size_t)n, f) == (size_t)n;
}
template <class F>
bool fields(Symbolic& S, double& cap, F&& io) {
  return io.sc(S.n) && io.sc(S.nnzA) && io.sc(S.nnzL) && io.sc(S.flops_exact) && io.sc(S.added) && io.sc(S.nmerges) &&
         io.sc(S.nsuper) && io.sc(S.nlevels) && io.sc(cap) && io.v(S.post) && io.v(S.parent3) && io.v(S.cc3) &&
         io.v(S.ffirst) && io.v(S.fparent) && io.v(S.fgroup) && io.v(S.perm_final) && io.v(S.iperm_final) &&
         io.v(S.sfirst) && io.v(S.sparent) && io.v(S.snode) && io.v(S.rows_ptr) && io.v(S.rows) && io.v(S.rel_ptr) &&
         io.v(S.rel_off) && io.v(S.rel_anc) && io.v(S.rel_q0) && io.v(S.relind) && io.v(S.parent_final) &&
         io.v(S.cc_final) && io.v(S.blk_ptr) && io.v(S.blk_q) && io.v(S.blk_len) && io.v(S.blk_anc) &&
         io.v(S.blk_relind) && io.v(S.level) && io.v(S.a_col) && io.v(S.a_pos);
}
struct Writer {
  FILE* f;
  template <class T> bool sc(const T& x) { return fwrite(&x, sizeof x, 1, f) == 1; }
  template <class T> bool v(const std::vector<T>& x) { return wvec(f, x); }
};
struct Reader {
  FILE* f;
  template <class T> bool sc(T& x) { return fread(&x, sizeof x, 1, f) == 1; }
  template <class T> bool v(std::vector<T>& x) { return rvec(f, x); }
};
// Consistency of a deserialised analysis before anything indexes with it: array lengths against
// n / nsuper / nnzA, monotone pointer arrays with the right final values, every index in range.
bool valid_symbolic(const Symbolic& S, std::string& why) {
  const int64_t n = S.n, ns = S.nsuper;
  auto bad = [&](const char* w) { why = w; return false; };
  if (n < 1 || n > INT32_MAX || ns < 1 || ns > n || S.nnzA < n || S.nlevels < 1 || S.nlevels > ns) return bad("scalars");
  auto len = [](const auto& v, int64_t x) { return (int64_t)v.size() == x; };
  if (!len(S.post, n) || !len(S.parent3, n) || !len(S.cc3, n) || !len(S.perm_final, n) || !len(S.iperm_final, n) ||
      !len(S.parent_final, n) || !len(S.cc_final, n) || !len(S.snode, n) || !len(S.sfirst, ns + 1) ||
      !len(S.sparent, ns) || !len(S.rows_ptr, ns + 1) || !len(S.rel_ptr, ns + 1) || !len(S.level, ns) ||
      !len(S.blk_ptr, ns + 1) || !len(S.a_col, S.nnzA) || !len(S.a_pos, S.nnzA))
    return bad("array lengths");
  auto in = [](int64_t v, int64_t lo, int64_t hi) { return v >= lo && v < hi; };
  std::vector<char> seen(n, 0);
  for (int64_t i = 0; i < n; ++i) {
    if (!in(S.perm_final[i], 0, n) || seen[S.perm_final[i]]) return bad("perm_final is not a permutation");
    seen[S.perm_final[i]] = 1;
    if (S.iperm_final[S.perm_final[i]] != i) return bad("iperm_final");
    if (!in(S.snode[i], 0, ns) || !(S.parent_final[i] == -1 || in(S.parent_final[i], i + 1, n))) return bad("snode / parent");
  }
  if (S.sfirst[0] != 0 || S.sfirst[ns] != n || S.rows_ptr[0] != 0 || (int64_t)S.rows.size() != S.rows_ptr[ns] ||
      S.rel_ptr[0] != 0 || (int64_t)S.rel_anc.size() != S.rel_ptr[ns] || !len(S.rel_q0, S.rel_ptr[ns]) ||
      !len(S.rel_off, S.rel_ptr[ns] + 1) || S.blk_ptr[0] != 0 || !len(S.blk_q, S.blk_ptr[ns]) ||
      !len(S.blk_len, S.blk_ptr[ns]) || !len(S.blk_anc, S.blk_ptr[ns]) || !len(S.blk_relind, S.blk_ptr[ns]))
    return bad("pointer ends");
  for (int64_t J = 0; J < ns; ++J) {
    const int64_t k = S.sfirst[J + 1] - S.sfirst[J], m = S.rows_ptr[J + 1] - S.rows_ptr[J];
    if (k < 1 || m < k || m > n || S.rel_ptr[J + 1] < S.rel_ptr[J] || S.blk_ptr[J + 1] < S.blk_ptr[J]) return bad("supernode shape");
    if (!(S.sparent[J] == -1 || in(S.sparent[J], J + 1, ns)) || !in(S.level[J], 0, S.nlevels)) return bad("supernode tree");
    for (int64_t q = S.rows_ptr[J]; q < S.rows_ptr[J + 1]; ++q)
      if (!in(S.rows[q], 0, n) || (q > S.rows_ptr[J] && S.rows[q] <= S.rows[q - 1])) return bad("rows(J)");
    for (int64_t c = 0; c < k; ++c)
      if (S.rows[S.rows_ptr[J] + c] != S.sfirst[J] + c || S.snode[S.sfirst[J] + c] != J) return bad("rows(J) columns");
    for (int64_t p = S.rel_ptr[J]; p < S.rel_ptr[J + 1]; ++p) {
      if (!in(S.rel_anc[p], J + 1, ns) || !in(S.rel_q0[p], k, m)) return bad("relind pairs");
      const int64_t mP = S.rows_ptr[S.rel_anc[p] + 1] - S.rows_ptr[S.rel_anc[p]];
      if (S.rel_off[p + 1] < S.rel_off[p] || S.rel_off[p + 1] > (int64_t)S.relind.size()) return bad("rel_off");
      for (int64_t x = S.rel_off[p]; x < S.rel_off[p + 1]; ++x)
        if (!in(S.relind[x], 0, mP)) return bad("relind range");
    }
    for (int64_t b = S.blk_ptr[J]; b < S.blk_ptr[J + 1]; ++b)
      if (!in(S.blk_anc[b], J + 1, ns) || !in(S.blk_q[b], k, m) || S.blk_len[b] < 1 || S.blk_q[b] + S.blk_len[b] > m)
        return bad("RLB blocks");
  }
  if (S.rel_off.back() != (int64_t)S.relind.size()) return bad("relind length");
  for (int64_t e = 0; e < S.nnzA; ++e) {
    if (!in(S.a_col[e], 0, n)) return bad("a_col");
    const int32_t J = S.snode[S.a_col[e]];
    if (!in(S.a_pos[e], S.a_col[e] - S.sfirst[J], S.rows_ptr[J + 1] - S.rows_ptr[J])) return bad("a_pos");
  }
  return true;
}
}  // namespace

extern "C" int spchol_save_analysis(const spchol_handle* h, const char* path) {
  if (!h || !path) return fail(SPCHOL_ERR_VALIDATION, "NULL argument");
  FILE* f = fopen(path, "wb");
  if (!f) return fail(SPCHOL_ERR_VALIDATION, std::string("cannot open ") + path);
  double cap = h->opt.merge_cap;
  Writer w{f};
  bool ok = fwrite(&SPCHOL_MAGIC, 8, 1, f) == 1 && fwrite(&SPCHOL_FORMAT, 8, 1, f) == 1 &&
            fields(const_cast<Symbolic&>(h->S), cap, w);
  ok = (fclose(f) == 0) && ok;
  return ok ? SPCHOL_OK : fail(SPCHOL_ERR_VALIDATION, std::string("write failed: ") + path);
}

extern "C" int spchol_load_analysis(const char* path, const spchol_options* opt, spchol_handle** out) {
  if (!path || !out) return fail(SPCHOL_ERR_VALIDATION, "NULL argument");
  *out = nullptr;
  FILE* f = fopen(path, "rb");
  if (!f) return fail(SPCHOL_ERR_VALIDATION, std::string("cannot open ") + path);
  spchol_handle* h = new spchol_handle();
  if (opt) h->opt = *opt; else spchol_default_options(&h->opt);
  char uid[128];
  const bool attach = apply_dist_init(h->opt, uid);
  uint64_t magic = 0, fmt = 0;
  double cap = 0;
  Reader r{f};
  bool ok = fread(&magic, 8, 1, f) == 1 && fread(&fmt, 8, 1, f) == 1 && magic == SPCHOL_MAGIC && fmt == SPCHOL_FORMAT &&
            fields(h->S, cap, r);
  fclose(f);
  if (!ok) { delete h; return fail(SPCHOL_ERR_VALIDATION, std::string("not a spchol analysis file: ") + path); }
  std::string why;
  if (!valid_symbolic(h->S, why)) { delete h; return fail(SPCHOL_ERR_VALIDATION, std::string("inconsistent analysis file (") + why + "): " + path); }
  h->opt.merge_cap = cap;   // the analysis was built with this cap
  int rc = finish_handle(h);
  if (rc != SPCHOL_OK) { delete h; return rc; }
  if (attach && h->opt.device >= 0) {
    rc = spchol_dist_attach_nccl(h, uid);
    if (rc != SPCHOL_OK) { spchol_destroy(h); return rc; }
  }
  *out = h;
  return SPCHOL_OK;
}

static bool host_only(const spchol_handle* h) { return h->opt.device < 0; }

extern "C" int spchol_set_values(spchol_handle* h, const double* values) {
  if (!h || !values) return fail(SPCHOL_ERR_VALIDATION, "NULL handle or values");
  if (host_only(h)) return fail(SPCHOL_ERR_STATE, "host-only handle (device < 0)");
  CK(cudaSetDevice(h->opt.device));
  const bool zero = h->world == 1 && !h->capped && h->zstream;
  if (zero) {   // zero the arena on the side stream during the upload (after the handle's earlier work)
    CK(cudaEventRecord(h->ev_zs, h->stream));
    CK(cudaStreamWaitEvent(h->zstream, h->ev_zs, 0));
    CK(cudaMemsetAsync(h->d_panels, 0, sizeof(double) * (size_t)std::max(1LL, h->panel_doubles), h->zstream));
    CK(cudaEventRecord(h->ev_zd, h->zstream));
  }
  CK(cudaMemcpyAsync(h->d_avals, values, sizeof(double) * (size_t)h->S.nnzA, cudaMemcpyHostToDevice, h->stream));
  if (zero) CK(cudaStreamWaitEvent(h->stream, h->ev_zd, 0));
  CK(cudaStreamSynchronize(h->stream));
  h->values_set = true;
  h->factored = false;
  h->prezeroed = zero;
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

// Enqueue the plan entries [begin, end) (launches, lookahead fork/join events) on st.
static int enqueue_ops(spchol_handle* h, cudaStream_t st, size_t begin, size_t end) {
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
  // The plan's stream 0 (critical path) runs on a high-priority internal stream so its few-CTA
  // cdiv launches are scheduled ahead of the trailing-update CTAs of stream 1 (low priority).
  // Both fork from st and join back into it (required under graph capture).  With kernel
  // timing enabled everything runs serialized on st.
  const bool multi = !h->timing;
  std::vector<char> used(h->pstreams.size(), 0);
  for (size_t i = begin; i < end; ++i) used[h->plan[i].stream] = 1;
  used[0] = 1;
  if (multi) {
    CK(cudaEventRecord(h->ev_fork, st));
    for (size_t q = 0; q < used.size(); ++q)
      if (used[q]) CK(cudaStreamWaitEvent(h->pstreams[q], h->ev_fork, 0));
  }
  int cur_level = -2;
  for (size_t i = begin; i < end; ++i) {
    const Launch& L = h->plan[i];
    cudaStream_t ls = multi ? h->pstreams[L.stream] : st;
    if (i < h->plan_level.size() && h->plan_level[i] != cur_level) {   // one NVTX range per level
      if (cur_level != -2) nvtxRangePop();
      cur_level = h->plan_level[i];
      char nm[32];
      std::snprintf(nm, sizeof nm, "level %d", cur_level);
      nvtxRangePushA(nm);
    }
    if (L.op == OP_RECORD) {
      if (multi) CK(cudaEventRecord(h->plan_events[L.ev], ls));
      continue;
    }
    if (L.op == OP_WAIT) {
      if (multi) CK(cudaStreamWaitEvent(ls, h->plan_events[L.ev], 0));
      continue;
    }
    if (L.op == OP_EXCHANGE) {
      int rc = dist_enqueue_exchange(h, ls, L.aux);
      if (rc) return rc;
      continue;
    }
    if (L.op == OP_BCAST) {
      int rc = dist_enqueue_bcast(h, ls, L.aux, L.aux2);
      if (rc) return rc;
      continue;
    }
    size_t ti = tstart((int)i);
    const bool hi = !(L.stream & 1) || (L.kind == K_LOCAL && L.aux == 1);   // NEXT_b: high priority on stream 1
    const int prio = multi ? (hi ? h->prio_hi : h->prio_lo) : 0;
    switch (L.kind) {
      case K_RLB:
        launch_rlb(h->d_rtasks + L.off, L.n, h->d_sn, h->d_panels, ls, prio);
        break;
      case K_SMALL:
        launch_small(h->d_small_sns + L.off, L.n, h->d_sn, h->d_sfirst, h->d_panels, h->d_ucol_base, h->d_ucol_map,
                     h->d_posmap, h->d_fail, L.aux, L.aux2, h->opt.deterministic ? 1 : 0, ls, prio, L.aux3);
        break;
      case K_POTRF:
        launch_potrf(h->d_ptasks + L.off, L.n, h->d_sn, h->d_sfirst, h->d_panels, h->d_linv, h->d_fail, ls, prio);
        break;
      case K_PANEL:
        launch_panel(h->d_pantasks + L.off, L.aux2, L.n - L.aux2, h->d_pansync + h->npanflags + 3 * L.aux, h->d_pansync,
                     h->d_sn, h->d_sfirst, h->d_panels, h->d_linv, h->d_fail, h->panel_grid, ls, prio, h->npanflags,
                     h->world > 1 ? INT_MAX : h->nslots_total);
        break;
      case K_TRSM:
        if (h->use_tma)
          launch_gemm_tma(MODE_TRSM, h->d_gtasks + L.off, L.n, h->d_sn, h->d_panels, h->d_tmaps, h->d_tmap_linv, h->d_ucol_base, h->d_ucol_map, h->d_posmap, ls, prio);
        else
          launch_gemm(MODE_TRSM, h->d_gtasks + L.off, L.n, h->d_sn, h->d_panels, h->d_linv, h->d_ucol_base, h->d_ucol_map, h->d_posmap, ls, prio);
        break;
      case K_LOCAL:
        if (h->use_tma)
          launch_gemm_tma(MODE_LOCAL, h->d_gtasks + L.off, L.n, h->d_sn, h->d_panels, h->d_tmaps, h->d_tmap_linv, h->d_ucol_base, h->d_ucol_map, h->d_posmap, ls, prio);
        else   // trailing-stream updates may reserve extra shared memory to cap their CTAs per SM
          launch_gemm(MODE_LOCAL, h->d_gtasks + L.off, L.n, h->d_sn, h->d_panels, h->d_linv, h->d_ucol_base, h->d_ucol_map, h->d_posmap, ls, prio,
                      multi && !hi ? h->rest_smem : 0);
        break;
      case K_SCATTER:
        if (L.aux == 2) {   // multi-GPU: partial U_J over the owned block columns
          int lw = 0;
          while ((1 << lw) < h->outer * h->nb) ++lw;
          launch_gemm(MODE_SCATTER_KS, h->d_gtasks + L.off, L.n, h->d_sn, h->d_panels, h->d_linv, h->d_ucol_base,
                      h->d_ucol_map, h->d_posmap, ls, prio, 0, lw);
        } else if (L.aux == 1)
          launch_gemm(MODE_SCATTER_DET, h->d_gtasks + L.off, L.n, h->d_sn, h->d_panels, h->d_linv, h->d_ucol_base, h->d_ucol_map, h->d_posmap, ls, prio);
        else if (h->use_tma)
          launch_gemm_tma(MODE_SCATTER, h->d_gtasks + L.off, L.n, h->d_sn, h->d_panels, h->d_tmaps, h->d_tmap_linv, h->d_ucol_base, h->d_ucol_map, h->d_posmap, ls, prio);
        else
          launch_gemm(MODE_SCATTER, h->d_gtasks + L.off, L.n, h->d_sn, h->d_panels, h->d_linv, h->d_ucol_base, h->d_ucol_map, h->d_posmap, ls, prio);
        break;
    }
    tstop(ti);
  }
  if (cur_level != -2) nvtxRangePop();
  if (multi) {   // join every stream the range used back into st (required under capture)
    for (size_t q = 0; q < used.size(); ++q)
      if (used[q]) {
        CK(cudaEventRecord(h->join_events[q], h->pstreams[q]));
        CK(cudaStreamWaitEvent(st, h->join_events[q], 0));
      }
  }
  CK(cudaGetLastError());
  return SPCHOL_OK;
}

// a1: fail flag reset, panels := 0, A's entries (this rank's share under multi-GPU) into the arena.
static int enqueue_init(spchol_handle* h, cudaStream_t st) {
  size_t ti = 0;
  if (h->timing) {
    while (h->ev_used + 2 > h->ev_pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      h->ev_pool.push_back(e);
    }
    ti = h->ev_used;
    h->ev_used += 2;
    cudaEventRecord(h->ev_pool[ti], st);
    h->pending.push_back({-1, ti});
  }
  if (h->world > 1) {
    int rc = dist_enqueue_init(h, st);
    if (rc) return rc;
  } else {
    CK(cudaMemsetAsync(h->d_fail, 0xFF, sizeof(unsigned long long), st));
    if (!h->skip_zero)   // (else zeroed by spchol_set_values alongside the upload)
      CK(cudaMemsetAsync(h->d_panels, 0, sizeof(double) * (size_t)std::max(1LL, h->panel_doubles), st));
    launch_init(h->d_avals, h->d_amap, h->S.nnzA, h->d_panels, st);
  }
  if (h->timing) cudaEventRecord(h->ev_pool[ti + 1], st);
  CK(cudaGetLastError());
  return SPCHOL_OK;
}

// Memory-capped factor: the top's entries once; per batch: window zeroed, the batch's entries, its
// levels, its finished panels to the host copy (stream-ordered, so the next batch's memset waits for
// the copy); then the resident top.
static int enqueue_factor_capped(spchol_handle* h, cudaStream_t st) {
  CK(cudaMemsetAsync(h->d_fail, 0xFF, sizeof(unsigned long long), st));
  CK(cudaMemsetAsync(h->d_panels + h->top_base, 0, sizeof(double) * (size_t)(h->panel_doubles - h->top_base), st));
  const int nb = h->nbatch;
  launch_init_list(h->d_avals, h->d_ainit_idx + h->ainit_off[nb], h->d_ainit_dst + h->ainit_off[nb],
                   h->ainit_off[nb + 1] - h->ainit_off[nb], h->d_panels, st);
  for (int b = 0; b < nb; ++b) {
    CK(cudaMemsetAsync(h->d_panels, 0, sizeof(double) * (size_t)h->batch_len[b], st));
    launch_init_list(h->d_avals, h->d_ainit_idx + h->ainit_off[b], h->d_ainit_dst + h->ainit_off[b],
                     h->ainit_off[b + 1] - h->ainit_off[b], h->d_panels, st);
    int rc = enqueue_ops(h, st, h->plan_batch[b], h->plan_batch[b + 1]);
    if (rc) return rc;
    CK(cudaMemcpyAsync(h->h_panels + h->batch_host[b], h->d_panels, sizeof(double) * (size_t)h->batch_len[b],
                       cudaMemcpyDeviceToHost, st));
  }
  int rc = enqueue_ops(h, st, h->plan_batch[nb], h->plan_all_end);
  if (rc) return rc;
  CK(cudaGetLastError());
  return SPCHOL_OK;
}

static int enqueue_factor(spchol_handle* h, cudaStream_t st) {
  // panel_kernel ready flags and tickets start at 0 in every factor
  if (h->npanflags + h->npanlaunch > 0)
    CK(cudaMemsetAsync(h->d_pansync, 0, sizeof(int) * ((size_t)h->npanflags + 3 * (size_t)h->npanlaunch), st));
  if (h->capped) return enqueue_factor_capped(h, st);
  int rc = enqueue_init(h, st);
  if (rc) return rc;
  if (h->world == 1) return enqueue_ops(h, st, h->plan_factor_begin, h->plan_all_end);
  if (!h->nccl_comm) return fail(SPCHOL_ERR_STATE, "multi-GPU handle without an NCCL communicator (spchol_dist_attach_nccl)");
  if ((rc = enqueue_ops(h, st, h->plan_all_end, h->plan_a_end))) return rc;   // phase A: own subtrees
  // exchange of the boundary blocks, then phase C (top levels with their broadcasts and exchanges)
  if ((rc = enqueue_ops(h, st, h->plan_a_end, h->plan.size()))) return rc;
  CK(cudaEventRecord(h->ev_comm_out, h->comm_stream));   // join the comm stream (graph capture)
  CK(cudaStreamWaitEvent(st, h->ev_comm_out, 0));
  int r = g_nccl.allreduce(h->d_fail, h->d_fail, 1, NCCL_UINT64, NCCL_MIN, h->nccl_comm, st);
  if (r) return nccl_fail(r, "ncclAllReduce(fail flag)");
  return SPCHOL_OK;
}

extern "C" int spchol_factor_async(spchol_handle* h) {
  Nvtx nv("spchol_factor");
  if (!h) return fail(SPCHOL_ERR_VALIDATION, "NULL handle");
  if (host_only(h)) return fail(SPCHOL_ERR_STATE, "host-only handle (device < 0)");
  if (!h->values_set) return fail(SPCHOL_ERR_STATE, "values not set");
  CK(cudaSetDevice(h->opt.device));
  h->factored = false;
  // multi-GPU: the NCCL calls are captured with the kernels (NCCL supports stream capture) from the
  // second factor on — the first runs eagerly so that NCCL sets up its peer connections outside a
  // capture; if the capture fails the handle stays eager.  The tests' blocking stand-in is never
  // captured.
  const bool dist_graph = h->world > 1 && g_nccl.capturable && !h->dist_capture_failed && h->dist_eager_done &&
                          !(getenv("SPCHOL_DIST_GRAPH") && atoi(getenv("SPCHOL_DIST_GRAPH")) == 0);
  // the arena was zeroed by spchol_set_values: this factor skips its memset (variant graph)
  h->skip_zero = h->prezeroed && h->world == 1 && !h->capped;
  h->prezeroed = false;
  if (h->skip_zero && h->opt.use_graph && !h->timing) {
    int rc = SPCHOL_OK;
    if (!h->gexec_nz) {
      cudaStream_t cs = h->own_stream;
      CK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
      rc = enqueue_factor(h, cs);
      cudaGraph_t g = nullptr;
      cudaError_t e = cudaStreamEndCapture(cs, &g);
      if (rc != SPCHOL_OK || e != cudaSuccess) {
        if (g) cudaGraphDestroy(g);
        h->skip_zero = false;
        return rc != SPCHOL_OK ? rc : cuda_fail(e, "cudaStreamEndCapture");
      }
      h->graph_nz = g;
      CK(cudaGraphInstantiateWithFlags(&h->gexec_nz, g, cudaGraphInstantiateFlagUseNodePriority));
    }
    h->skip_zero = false;
    CK(cudaGraphLaunch(h->gexec_nz, h->stream));
    return SPCHOL_OK;
  }
  if (h->skip_zero) {   // eager (no graph / kernel timing)
    const int rc = enqueue_factor(h, h->stream);
    h->skip_zero = false;
    return rc;
  }
  if (h->opt.use_graph && !h->timing && (h->world == 1 || dist_graph)) {
    if (!h->gexec) {
      cudaStream_t cs = h->own_stream;
      CK(cudaStreamBeginCapture(cs, h->world > 1 ? cudaStreamCaptureModeRelaxed : cudaStreamCaptureModeThreadLocal));
      int rc = enqueue_factor(h, cs);
      cudaGraph_t g = nullptr;
      cudaError_t e = cudaStreamEndCapture(cs, &g);
      if (h->world > 1 && (rc != SPCHOL_OK || e != cudaSuccess)) {   // stay eager (NCCL refused the capture)
        if (g) cudaGraphDestroy(g);
        cudaGetLastError();
        h->dist_capture_failed = true;
        return enqueue_factor(h, h->stream);
      }
      if (rc != SPCHOL_OK) { if (g) cudaGraphDestroy(g); return rc; }
      if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture");
      h->graph = g;
      CK(cudaGraphInstantiateWithFlags(&h->gexec, g, cudaGraphInstantiateFlagUseNodePriority));  // honour per-node priorities
      h->graph_dist = h->world > 1;
    }
    CK(cudaGraphLaunch(h->gexec, h->stream));
    return SPCHOL_OK;
  }
  h->dist_eager_done = true;
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
// the CTA).  Large supernodes: one launch per level and direction (solve_fwd/bwd_level_kernel):
// 64-row / 64-column block tasks that wait on per-block ready flags instead of kernel boundaries;
// the diagonal blocks are applied with the inverses kept from the factor (X_bb = L_bb^{-1}).
// Memory-capped solve: forward batch by batch (each copied back into the window), then the resident
// top; backward the top, then the batches in reverse (copied back again).
static int enqueue_solve_capped(spchol_handle* h, const double* d_b, double* d_x, int nr, cudaStream_t st) {
  const Symbolic& S = h->S;
  launch_permute(h->d_perm, d_b, h->d_y, S.n, nr, 0, st);
  const size_t NS = (size_t)std::max(1, h->nslots_total);
  int* fflag = h->d_sflags;
  int* bflag = fflag + NS;
  int* rcnt = bflag + NS;
  int* tickets = rcnt + NS;
  CK(cudaMemsetAsync(h->d_sflags, 0, sizeof(int) * (3 * NS + h->nticket), st));
  const int nseg = (int)h->segs.size(), nl = S.nlevels;
  auto fwd = [&](int g) {
    const auto& G = h->segs[g];
    for (int l = 0; l < nl; ++l) {
      for (int cl = 0; cl < 3; ++cl)
        launch_solve_small(h->d_ssolve + G.ss[3 * l + cl], G.ss[3 * l + cl + 1] - G.ss[3 * l + cl], cl, 0, h->d_rows,
                           h->d_panels, h->d_y, nr, st);
      launch_solve_fwd_level(h->d_stasks + G.fwd[l], (int)(G.bwd[l] - G.fwd[l]), tickets + 2 * (g * nl + l), fflag,
                             h->d_sn, h->d_sfirst, h->d_rows_ptr, h->d_rows, h->d_panels, h->d_linv, h->d_y, h->nb, nr, st);
    }
  };
  auto bwd = [&](int g) {
    const auto& G = h->segs[g];
    for (int l = nl - 1; l >= 0; --l) {
      launch_solve_bwd_level(h->d_stasks + G.bwd[l], (int)(G.fwd[l + 1] - G.bwd[l]), tickets + 2 * (g * nl + l) + 1,
                             bflag, rcnt, h->d_sn, h->d_sfirst, h->d_rows_ptr, h->d_rows, h->d_panels, h->d_linv, h->d_y,
                             h->nb, nr, st);
      for (int cl = 0; cl < 3; ++cl)
        launch_solve_small(h->d_ssolve + G.ss[3 * l + cl], G.ss[3 * l + cl + 1] - G.ss[3 * l + cl], cl, 1, h->d_rows,
                           h->d_panels, h->d_y, nr, st);
    }
  };
  for (int b = 0; b < h->nbatch; ++b) {
    CK(cudaMemcpyAsync(h->d_panels, h->h_panels + h->batch_host[b], sizeof(double) * (size_t)h->batch_len[b],
                       cudaMemcpyHostToDevice, st));
    fwd(b);
  }
  fwd(nseg - 1);
  bwd(nseg - 1);
  for (int b = h->nbatch - 1; b >= 0; --b) {
    CK(cudaMemcpyAsync(h->d_panels, h->h_panels + h->batch_host[b], sizeof(double) * (size_t)h->batch_len[b],
                       cudaMemcpyHostToDevice, st));
    bwd(b);
  }
  launch_permute(h->d_perm, h->d_y, d_x, S.n, nr, 1, st);
  CK(cudaGetLastError());
  return SPCHOL_OK;
}

static int enqueue_solve(spchol_handle* h, const double* d_b, double* d_x, int nr, cudaStream_t st) {
  if (h->capped) return enqueue_solve_capped(h, d_b, d_x, nr, st);
  const Symbolic& S = h->S;
  launch_permute(h->d_perm, d_b, h->d_y, S.n, nr, 0, st);
  const size_t NS = (size_t)std::max(1, h->nslots_total);
  int* fflag = h->d_sflags;
  int* bflag = fflag + NS;
  int* rcnt = bflag + NS;
  int* tickets = rcnt + NS;
  CK(cudaMemsetAsync(h->d_sflags, 0, sizeof(int) * (3 * NS + 2 * (size_t)S.nlevels + 1), st));
  for (int l = 0; l < S.nlevels; ++l) {
    for (int cl = 0; cl < 3; ++cl)
      launch_solve_small(h->d_ssolve + h->ssolve_off[3 * l + cl], h->ssolve_off[3 * l + cl + 1] - h->ssolve_off[3 * l + cl],
                         cl, 0, h->d_rows, h->d_panels, h->d_y, nr, st);
    launch_solve_fwd_level(h->d_stasks + h->sfwd_off[l], (int)(h->sbwd_off[l] - h->sfwd_off[l]), tickets + 2 * l, fflag,
                           h->d_sn, h->d_sfirst, h->d_rows_ptr, h->d_rows, h->d_panels, h->d_linv, h->d_y, h->nb, nr, st);
  }
  for (int l = S.nlevels - 1; l >= 0; --l) {
    launch_solve_bwd_level(h->d_stasks + h->sbwd_off[l], (int)(h->sfwd_off[l + 1] - h->sbwd_off[l]), tickets + 2 * l + 1,
                           bflag, rcnt, h->d_sn, h->d_sfirst, h->d_rows_ptr, h->d_rows, h->d_panels, h->d_linv, h->d_y,
                           h->nb, nr, st);
    for (int cl = 0; cl < 3; ++cl)
      launch_solve_small(h->d_ssolve + h->ssolve_off[3 * l + cl], h->ssolve_off[3 * l + cl + 1] - h->ssolve_off[3 * l + cl],
                         cl, 1, h->d_rows, h->d_panels, h->d_y, nr, st);
  }
  launch_permute(h->d_perm, h->d_y, d_x, S.n, nr, 1, st);
  CK(cudaGetLastError());
  return SPCHOL_OK;
}

// One solve of the internal buffer d_y2 in place, captured in a CUDA graph on first use.
// Multi-GPU: the distributed solve (dist_enqueue_solve) is collective — every rank of the handle's
// communicator calls the solve the same number of times (and with the same nrhs).
static int any_solve(spchol_handle* h, int nr, cudaStream_t st) {
  return h->world > 1 ? dist_enqueue_solve(h, h->d_y2, nr, st) : enqueue_solve(h, h->d_y2, h->d_y2, nr, st);
}
// One solve of the nr right-hand sides staged in d_y2 (column-major, ld n), in place; captured in a
// CUDA graph per nr on first use.
static int run_solve_y2(spchol_handle* h, int nr) {
  // multi-GPU: captured from the second solve on, as the factor
  const bool graph = h->opt.use_graph &&
                     (h->world == 1 || (g_nccl.capturable && h->dist_solve_eager_done && !h->dist_capture_failed));
  h->dist_solve_eager_done = true;
  if (!graph) return any_solve(h, nr, h->stream);
  const int gi = nr == 4 ? 2 : nr == 2 ? 1 : 0;
  if (!h->solve_gexec[gi]) {
    cudaStream_t cs = h->own_stream;
    CK(cudaStreamBeginCapture(cs, h->world > 1 ? cudaStreamCaptureModeRelaxed : cudaStreamCaptureModeThreadLocal));
    int rc = any_solve(h, nr, cs);
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamEndCapture(cs, &g);
    if (h->world > 1 && (rc != SPCHOL_OK || e != cudaSuccess)) {   // stay eager (NCCL refused the capture)
      if (g) cudaGraphDestroy(g);
      cudaGetLastError();
      h->dist_capture_failed = true;
      return any_solve(h, nr, h->stream);
    }
    if (rc != SPCHOL_OK) { if (g) cudaGraphDestroy(g); return rc; }
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture(solve)");
    h->solve_graph[gi] = g;
    CK(cudaGraphInstantiateWithFlags(&h->solve_gexec[gi], g, 0));
  }
  CK(cudaGraphLaunch(h->solve_gexec[gi], h->stream));
  return SPCHOL_OK;
}

// nrhs right-hand sides in blocks of 4, 2, 1 (each block one pass over L).
static int solve_blocks(spchol_handle* h, const double* b, double* x, int32_t nrhs, int64_t ld, cudaMemcpyKind kin,
                        cudaMemcpyKind kout) {
  Nvtx nv("spchol_solve");
  const size_t n = (size_t)h->S.n;
  for (int r0 = 0; r0 < nrhs;) {
    const int left = nrhs - r0, nr = left >= 4 ? 4 : left >= 2 ? 2 : 1;
    CK(cudaMemcpy2DAsync(h->d_y2, n * sizeof(double), b + (size_t)r0 * ld, (size_t)ld * sizeof(double), n * sizeof(double),
                         nr, kin, h->stream));
    int rc = run_solve_y2(h, nr);
    if (rc != SPCHOL_OK) return rc;
    CK(cudaMemcpy2DAsync(x + (size_t)r0 * ld, (size_t)ld * sizeof(double), h->d_y2, n * sizeof(double), n * sizeof(double),
                         nr, kout, h->stream));
    r0 += nr;
  }
  return SPCHOL_OK;
}

extern "C" int spchol_solve_device(spchol_handle* h, const double* d_b, double* d_x, int32_t nrhs, int64_t ld,
                                   void* stream) {
  if (!h) return fail(SPCHOL_ERR_VALIDATION, "NULL handle");
  if (host_only(h) || !h->factored) return fail(SPCHOL_ERR_STATE, "solve before a successful factor");
  if (nrhs < 1 || ld < h->S.n) return fail(SPCHOL_ERR_DIMENSION, "nrhs < 1 or ld < n");
  CK(cudaSetDevice(h->opt.device));
  cudaStream_t keep = h->stream;
  if (stream) h->stream = (cudaStream_t)stream;
  const int rc = solve_blocks(h, d_b, d_x, nrhs, ld, cudaMemcpyDeviceToDevice, cudaMemcpyDeviceToDevice);
  h->stream = keep;
  return rc;
}

extern "C" int spchol_solve(spchol_handle* h, const double* b, double* x, int32_t nrhs, int64_t ld) {
  if (!h) return fail(SPCHOL_ERR_VALIDATION, "NULL handle");
  if (host_only(h) || !h->factored) return fail(SPCHOL_ERR_STATE, "solve before a successful factor");
  if (nrhs < 1 || ld < h->S.n) return fail(SPCHOL_ERR_DIMENSION, "nrhs < 1 or ld < n");
  CK(cudaSetDevice(h->opt.device));
  int rc = solve_blocks(h, b, x, nrhs, ld, cudaMemcpyHostToDevice, cudaMemcpyDeviceToHost);
  if (rc) return rc;
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
    case SPCHOL_Q_PANEL_DOUBLES: *value = h->panel_off.empty() ? h->panel_doubles : h->panel_off.back(); break;
    case SPCHOL_Q_NMERGES: *value = S.nmerges; break;
    case SPCHOL_Q_FLOPS_EXACT: *value = (int64_t)S.flops_exact; break;
    case SPCHOL_Q_FLOPS_EXEC: *value = (int64_t)h->flops_exec; break;
    case SPCHOL_Q_LAUNCHES: {   // kernels one factor launches (init + the executed plan range)
      int64_t nl = 1;
      const size_t b = h->world == 1 ? h->plan_factor_begin : h->plan_all_end;
      const size_t e = h->world == 1 ? h->plan_all_end : h->plan.size();
      for (size_t i = b; i < e; ++i)   // a fused cdiv step launches the diagonal and (if any) the below kernel
        nl += h->plan[i].op == OP_LAUNCH ? (h->plan[i].kind == K_PANEL && h->plan[i].n > h->plan[i].aux2 ? 2 : 1) : 0;
      *value = nl;
      break;
    }
    case SPCHOL_Q_UPDATE_ENTRIES: *value = (int64_t)h->update_entries; break;
    case SPCHOL_Q_NBLOCKS: *value = (int64_t)S.blk_q.size(); break;
    case SPCHOL_Q_NMARKERS: *value = (int64_t)h->markers.size(); break;
    case SPCHOL_Q_DEVICE_BYTES: *value = (int64_t)h->device_bytes; break;
    case SPCHOL_Q_COMM_SEND_BYTES: *value = (int64_t)h->comm_send; break;
    case SPCHOL_Q_COMM_RECV_BYTES: *value = (int64_t)h->comm_recv; break;
    case SPCHOL_Q_ARENA_BYTES: {   // physical memory of this rank's panel arena + inverses (+ ring)
      if (h->world == 1) { *value = (int64_t)(8 * (h->panel_doubles + (long long)h->nslots_total * NBMAX * NBMAX)); break; }
      long long b = h->ring_bytes;
      for (const VRegion& g : h->vregions) if (g.ring < 0) b += 8 * g.len;
      const int r = h->rank, P = h->world;
      b += 8LL * NBMAX * NBMAX * ((h->slot_sub[r + 1] - h->slot_sub[r]) + (h->nslots_total - h->slot_sub[P]));
      *value = b;
      break;
    }
    case SPCHOL_Q_DIST_GRAPH: *value = h->graph_dist ? 1 : 0; break;
    case SPCHOL_Q_COMM_B_SEND_BYTES: *value = (int64_t)h->comm_b_send; break;
    case SPCHOL_Q_NBATCHES: *value = h->capped ? h->nbatch : 0; break;
    case SPCHOL_Q_HOST_BYTES: *value = h->capped ? 8 * (int64_t)h->batch_host[h->nbatch] : 0; break;
    case SPCHOL_Q_COMM_B_RECV_BYTES: *value = (int64_t)h->comm_b_recv; break;
    case SPCHOL_Q_NTOP_DIST: {
      int64_t c = 0;
      for (char d : h->top_dist) c += d != 0;
      *value = c;
      break;
    }
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

extern "C" int spchol_export_blocks(const spchol_handle* h, int64_t* blk_ptr, int32_t* blk_q, int32_t* blk_len,
                                    int32_t* blk_anc, int32_t* blk_relind) {
  if (!h) return fail(SPCHOL_ERR_VALIDATION, "NULL handle");
  const Symbolic& S = h->S;
  cp<int64_t>(blk_ptr, S.blk_ptr); cp(blk_q, S.blk_q); cp(blk_len, S.blk_len); cp(blk_anc, S.blk_anc);
  cp(blk_relind, S.blk_relind);
  return SPCHOL_OK;
}

// Panel J to host memory.  Multi-GPU: the entries this rank holds (its subtrees, the top supernodes
// it factors whole, its block columns of the distributed ones), zeros elsewhere — the sum over the
// ranks' exports is L.
static int copy_panel(const spchol_handle* h, int J, double* out) {
  const SnInfo& I = h->sn[J];
  const size_t cnt = (size_t)I.ld * I.k;
  if (!cnt) return SPCHOL_OK;
  const double* src = h->d_panels + I.off;
  if (h->capped && h->batch[J] >= 0) {   // a finished batch: its host copy
    std::memcpy(out, h->h_panels + h->host_off[J], sizeof(double) * cnt);
    return SPCHOL_OK;
  }
  if (h->world == 1) {
    CK(cudaMemcpy(out, src, sizeof(double) * cnt, cudaMemcpyDeviceToHost));
    return SPCHOL_OK;
  }
  std::fill(out, out + cnt, 0.0);
  const int W = outer_w(h);
  if (!h->top_dist[J]) {
    if (dist_owns(h, J, h->S.sfirst[J])) CK(cudaMemcpy(out, src, sizeof(double) * cnt, cudaMemcpyDeviceToHost));
    return SPCHOL_OK;
  }
  for (int C = 0; C * W < I.k; ++C)
    if (blk_owner(h, J, C) == h->rank) {
      const size_t o = (size_t)C * W * I.ld;
      CK(cudaMemcpy(out + o, src + o, sizeof(double) * (size_t)I.ld * std::min(W, I.k - C * W), cudaMemcpyDeviceToHost));
    }
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
  if (panels && h->panel_doubles > 0) {
    if (h->world == 1 && !h->capped) {
      CK(cudaMemcpy(panels, h->d_panels, sizeof(double) * (size_t)h->panel_doubles, cudaMemcpyDeviceToHost));
    } else {
      std::fill(panels, panels + h->panel_off.back(), 0.0);
      for (int J = 0; J < h->S.nsuper; ++J) {
        int rc = copy_panel(h, J, panels + h->panel_off[J]);
        if (rc) return rc;
      }
    }
  }
  return SPCHOL_OK;
}

extern "C" int spchol_export_panel(const spchol_handle* h, int32_t J, double* out) {
  if (!h || !out) return fail(SPCHOL_ERR_VALIDATION, "NULL argument");
  if (host_only(h)) return fail(SPCHOL_ERR_STATE, "host-only handle (device < 0)");
  if (J < 0 || J >= h->S.nsuper) return fail(SPCHOL_ERR_DIMENSION, "supernode index out of range");
  CK(cudaSetDevice(h->opt.device));
  CK(cudaStreamSynchronize(h->stream));
  return copy_panel(h, J, out);
}

// Exact factor in CSC (final numbering).  Pattern: struct(L_j) by row subtrees of the final etree
// (row i of L = the etree paths from every k < i with C_f(i,k) != 0 up to i); values
// from the panels, where the exact rows of column j are a subsequence of rows(snode(j)).
extern "C" int spchol_export_factor_csc(const spchol_handle* h, int64_t* Lp, int32_t* Li, double* Lx,
                                        int64_t* padding_nonzeros) {
  if (!h || !Lp) return fail(SPCHOL_ERR_VALIDATION, "NULL argument");
  if ((Lx || padding_nonzeros) && (host_only(h) || !h->factored))
    return fail(SPCHOL_ERR_STATE, "values need a successful factor on a device handle");
  const Symbolic& S = h->S;
  const int64_t n = S.n;
  Lp[0] = 0;
  for (int64_t j = 0; j < n; ++j) Lp[j + 1] = Lp[j] + S.cc_final[j];
  if (!Li && !Lx && !padding_nonzeros) return SPCHOL_OK;
  // lower C_f by rows: entry e of A sits at (final row, final col)
  std::vector<int64_t> rp(n + 1, 0);
  std::vector<int32_t> rrow(S.a_col.size());
  for (size_t e = 0; e < S.a_col.size(); ++e) {
    const int c = S.a_col[e], J = S.snode[c];
    rrow[e] = S.rows[S.rows_ptr[J] + S.a_pos[e]];
    if (rrow[e] > c) rp[rrow[e] + 1]++;
  }
  for (int64_t i = 0; i < n; ++i) rp[i + 1] += rp[i];
  std::vector<int32_t> rcol(rp[n]);
  {
    std::vector<int64_t> nx(rp.begin(), rp.end() - 1);
    for (size_t e = 0; e < S.a_col.size(); ++e)
      if (rrow[e] > S.a_col[e]) rcol[nx[rrow[e]]++] = S.a_col[e];
  }
  std::vector<int32_t> li(Lp[n]);
  std::vector<int64_t> nxt(Lp, Lp + n);
  std::vector<int32_t> mark(n, -1);
  for (int64_t i = 0; i < n; ++i) {
    mark[i] = (int32_t)i;
    li[nxt[i]++] = (int32_t)i;                       // diagonal first: rows ascend within a column
    for (int64_t e = rp[i]; e < rp[i + 1]; ++e)
      for (int32_t j = rcol[e]; mark[j] != i; j = S.parent_final[j]) {
        if (j < 0 || nxt[j] >= Lp[j + 1]) return fail(SPCHOL_ERR_VALIDATION, "row subtree inconsistent with cc");
        mark[j] = (int32_t)i;
        li[nxt[j]++] = (int32_t)i;
      }
  }
  for (int64_t j = 0; j < n; ++j)
    if (nxt[j] != Lp[j + 1]) return fail(SPCHOL_ERR_VALIDATION, "column count mismatch");
  if (Li) std::memcpy(Li, li.data(), sizeof(int32_t) * li.size());
  if (!Lx && !padding_nonzeros) return SPCHOL_OK;
  int64_t npad = 0;
  std::vector<double> panel;
  for (int J = 0; J < S.nsuper; ++J) {
    const SnInfo& I = h->sn[J];
    panel.resize((size_t)I.ld * I.k);
    int rc = spchol_export_panel(h, J, panel.data());
    if (rc != SPCHOL_OK) return rc;
    const int32_t* rJ = S.rows.data() + S.rows_ptr[J];
    for (int c = 0; c < I.k; ++c) {
      const int64_t j = S.sfirst[J] + c;
      int q = c;
      for (int64_t e = Lp[j]; e < Lp[j + 1]; ++e, ++q) {
        for (; q < I.m && rJ[q] != li[e]; ++q) npad += panel[(size_t)c * I.ld + q] != 0.0;
        if (q >= I.m) return fail(SPCHOL_ERR_VALIDATION, "exact row outside the panel");
        if (Lx) Lx[e] = panel[(size_t)c * I.ld + q];
      }
      for (; q < I.m; ++q) npad += panel[(size_t)c * I.ld + q] != 0.0;
    }
  }
  if (padding_nonzeros) *padding_nonzeros = npad;
  return SPCHOL_OK;
}

extern "C" int spchol_export_diagonal(spchol_handle* h, double* diag) {
  if (!h || !diag) return fail(SPCHOL_ERR_VALIDATION, "NULL argument");
  if (host_only(h)) return fail(SPCHOL_ERR_STATE, "host-only handle (device < 0)");
  CK(cudaSetDevice(h->opt.device));
  const Symbolic& S = h->S;
  if (h->capped) {   // the batches' panels live in the host copy
    CK(cudaStreamSynchronize(h->stream));
    std::vector<double> pan;
    for (int J = 0; J < S.nsuper; ++J) {
      pan.resize((size_t)h->sn[J].ld * h->sn[J].k);
      int rc = copy_panel(h, J, pan.data());
      if (rc) return rc;
      for (int c = 0; c < h->sn[J].k; ++c) diag[S.sfirst[J] + c] = pan[(size_t)c * h->sn[J].ld + c];
    }
    return SPCHOL_OK;
  }
  if (!h->d_diag_idx) {   // multi-GPU: the diagonal entries this rank holds, zeros elsewhere
    std::vector<long long> idx(S.n);
    for (int J = 0; J < S.nsuper; ++J)
      for (int c = 0; c < h->sn[J].k; ++c)
        idx[S.sfirst[J] + c] = h->world > 1 && !dist_owns(h, J, S.sfirst[J] + c)
                                   ? -1 : h->sn[J].off + (long long)c * h->sn[J].ld + c;
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

extern "C" int spchol_dist_nccl_unique_id(void* out128) {
  if (!out128) return fail(SPCHOL_ERR_VALIDATION, "NULL argument");
  std::string err;
  if (!nccl_load(err)) return fail(SPCHOL_ERR_NCCL, err);
  int r = g_nccl.getid(out128);
  return r ? nccl_fail(r, "ncclGetUniqueId") : SPCHOL_OK;
}

extern "C" int spchol_dist_attach_nccl(spchol_handle* h, const void* unique_id128) {
  if (!h || !unique_id128) return fail(SPCHOL_ERR_VALIDATION, "NULL argument");
  if (host_only(h)) return fail(SPCHOL_ERR_STATE, "host-only handle (device < 0)");
  if (h->nccl_comm) return fail(SPCHOL_ERR_STATE, "communicator already attached");
  std::string err;
  if (!nccl_load(err)) return fail(SPCHOL_ERR_NCCL, err);
  CK(cudaSetDevice(h->opt.device));
  NcclUid id;
  std::memcpy(id.internal, unique_id128, 128);
  void* comm = nullptr;
  int r = g_nccl.init(&comm, h->world, id, h->rank);
  if (r) return nccl_fail(r, "ncclCommInitRank");
  h->nccl_comm = comm;
  // one communicator per distinct top rank group smaller than the world (collective: every rank
  // calls ncclCommSplit for every group in the same order, members with colour 0, others without)
  std::vector<std::array<int, 2>> keys;
  for (int J = 0; J < h->S.nsuper; ++J)
    if (h->owner[J] < 0 && h->grp_hi[J] - h->grp_lo[J] < h->world) keys.push_back({h->grp_lo[J], h->grp_hi[J]});
  std::sort(keys.begin(), keys.end());
  keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
  h->grp_keys = keys;
  h->grp_comms.assign(keys.size(), nullptr);
  for (size_t i = 0; i < keys.size(); ++i) {
    const bool member = h->rank >= keys[i][0] && h->rank < keys[i][1];
    r = g_nccl.split(comm, member ? 0 : -1 /* NCCL_SPLIT_NOCOLOR */, h->rank, &h->grp_comms[i], nullptr);
    if (r) return nccl_fail(r, "ncclCommSplit(top rank group)");
  }
  return SPCHOL_OK;
}

extern "C" int spchol_export_mapping(const spchol_handle* h, int32_t* owner, int32_t* top_owner, int64_t* top_off,
                                     int64_t* top_slot) {
  if (!h) return fail(SPCHOL_ERR_VALIDATION, "NULL handle");
  if (owner) for (int J = 0; J < h->S.nsuper; ++J) owner[J] = h->world > 1 ? h->owner[J] : 0;
  if (top_owner) for (int J = 0; J < h->S.nsuper; ++J) top_owner[J] = h->world > 1 ? h->top_owner[J] : -1;
  if (top_off) *top_off = h->world > 1 ? h->sub_off[h->world] : h->panel_doubles;
  if (top_slot) *top_slot = h->world > 1 ? h->slot_sub[h->world] : h->nslots_total;
  return SPCHOL_OK;
}

extern "C" int spchol_dist_plan_flops(const spchol_handle* h, double* phase_a, double* top_level) {
  if (!h) return fail(SPCHOL_ERR_VALIDATION, "NULL handle");
  if (phase_a) *phase_a = 0;
  if (top_level) for (int l = 0; l < h->S.nlevels; ++l) top_level[l] = 0;
  if (h->world == 1) {
    if (phase_a) for (size_t i = h->plan_factor_begin; i < h->plan_all_end; ++i) if (h->plan[i].op == OP_LAUNCH) *phase_a += h->plan[i].flops;
    return SPCHOL_OK;
  }
  for (size_t i = h->plan_all_end; i < h->plan.size(); ++i) {
    const Launch& L = h->plan[i];
    if (L.op != OP_LAUNCH) continue;
    if (i < h->plan_a_end) { if (phase_a) *phase_a += L.flops; }
    else if (top_level) top_level[h->plan_level[i]] += L.flops;
  }
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
