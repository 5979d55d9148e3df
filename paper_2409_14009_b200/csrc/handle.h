// The spchol handle (include/spchol.h's opaque type): host symbolic data, launch plan, device
// layout in HBM.  Shared by capi.cu (plan, single-GPU drivers, C ABI) and dist.cu (multi-GPU).
// P:n = PAPER.md line n (arXiv 2409.14009).
#pragma once
#include <array>
#include <cstdint>
#include <string>
#include <vector>

#include <cuda.h>
#include <cuda_runtime.h>

#include "kernels.cuh"
#include "spchol.h"
#include "symbolic.h"

namespace spchol {

int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* where);
#define CK(call)                                                   \
  do {                                                             \
    cudaError_t e_ = (call);                                       \
    if (e_ != cudaSuccess) return ::spchol::cuda_fail(e_, #call);  \
  } while (0)

enum LaunchKind { K_SMALL = 0, K_POTRF = 1, K_TRSM = 2, K_LOCAL = 3, K_SCATTER = 4, K_INIT = 5, K_RLB = 6, K_PANEL = 7, K_NKINDS = 8 };

// NCCL, loaded on demand (dlopen of libnccl.so.2, normally the copy torch already loaded): the
// library has no link-time NCCL dependency and single-GPU use never touches it.
struct NcclUid { char internal[128]; };
typedef int (*nccl_getid_t)(void*);
typedef int (*nccl_init_t)(void**, int, NcclUid, int);
typedef int (*nccl_allreduce_t)(const void*, void*, size_t, int, int, void*, cudaStream_t);
typedef int (*nccl_reduce_t)(const void*, void*, size_t, int, int, int, void*, cudaStream_t);
typedef int (*nccl_p2p_t)(const void*, size_t, int, int, void*, cudaStream_t);
typedef int (*nccl_bcast_t)(const void*, void*, size_t, int, int, void*, cudaStream_t);
typedef int (*nccl_split_t)(void*, int, int, void**, void*);
typedef int (*nccl_group_t)();
typedef int (*nccl_destroy_t)(void*);
typedef const char* (*nccl_errstr_t)(int);
struct NcclApi {
  void* so = nullptr;
  nccl_getid_t getid = nullptr;
  nccl_init_t init = nullptr;
  nccl_allreduce_t allreduce = nullptr;
  nccl_reduce_t reduce = nullptr;
  nccl_p2p_t send = nullptr, recv = nullptr;
  nccl_bcast_t bcast = nullptr;
  nccl_split_t split = nullptr;
  nccl_group_t group_start = nullptr, group_end = nullptr;
  nccl_destroy_t destroy = nullptr;
  nccl_errstr_t errstr = nullptr;
  bool capturable = true;   // false for the tests' blocking single-process stand-in (tests/mock_nccl)
};
extern NcclApi g_nccl;
constexpr int NCCL_SUM = 0, NCCL_MIN = 3, NCCL_UINT64 = 5, NCCL_FLOAT64 = 8;
bool nccl_load(std::string& err);
int nccl_fail(int r, const char* where);

enum OpType { OP_LAUNCH = 0, OP_RECORD = 1, OP_WAIT = 2, OP_EXCHANGE = 3, OP_BCAST = 4 };
// One step of the factor's launch plan.  OP_LAUNCH: a batched kernel (kind, tasks [off, off+n)) on
// stream `stream` (even = critical path: cdiv chain + relind scatter, odd = trailing updates);
// OP_RECORD / OP_WAIT: event `ev` recorded on / awaited by `stream` (lookahead fork/join).
// Multi-GPU "markers" (every rank's plan holds the same sequence of them, so the NCCL calls pair up):
// OP_EXCHANGE (exchange aux): the update blocks of that exchange (after phase A: the subtrees'
// boundary blocks; after top level l: the partial U_J of the level's top supernodes) go to the
// owners of their destination block columns (grouped ncclSend/ncclRecv) and are extend-added there.
// OP_BCAST (distributed top supernode aux, outer block column aux2): the finished block column goes
// from its owner to the rest of the supernode's rank group (ncclBroadcast on the group communicator).
struct Launch {
  int kind;
  long long off;   // first task
  int n;           // tasks
  double flops, bytes;
  int op = OP_LAUNCH, stream = 0, ev = -1;
  int aux = 0;     // K_SMALL: dynamic shared memory (doubles); K_SCATTER: 1 = plain RMW (deterministic),
                   // 2 = K-split over owned block columns (multi-GPU)
  int aux2 = 0;    // K_SMALL: largest m in the launch
  int aux3 = 0;    // K_SMALL: largest k in the launch if it runs one warp per supernode, else 0
};

extern thread_local size_t g_dev_bytes;   // device bytes allocated by the handle being set up
template <class T>
cudaError_t dalloc(T** p, size_t count) {
  *p = nullptr;
  if (count == 0) count = 1;
  g_dev_bytes += count * sizeof(T);
  return cudaMalloc((void**)p, count * sizeof(T));
}
template <class T>
cudaError_t upload(T** p, const std::vector<T>& v) {
  cudaError_t e = dalloc(p, v.size());
  if (e != cudaSuccess) return e;
  if (!v.empty()) e = cudaMemcpy(*p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
  return e;
}

// Multi-GPU update block (dist.cu): a dense lower block over a sorted row set R (final numbering) —
// the boundary block of a subtree root S (R = R_S: every update its subtree sends above it lands in
// R_S x R_S, by containment P:172) or rank src's partial U_J of a top supernode J (R = R_J).  Its
// columns are cut into runs, one per destination (ancestor P, outer block column C): run = columns
// [j0, j1) x rows [j0, t) of R, stored column-major with leading dimension ld, so it is one
// contiguous message to the rank owning (P, C).
struct XBlk {
  int src, node, exch, kind;   // kind 0 = boundary block of subtree root node, 1 = partial U of top node
  int t;                       // |R|
  long long run0, run1;        // runs [run0, run1) in the global run list
};
struct XRun {
  int blk, j0, j1, P, C, dst;
  long long loc;    // offset (doubles) inside the source rank's update region
  long long roff;   // offset inside the destination rank's receive region (dst != src)
  int ld;
};
// A region of the per-rank arena (doubles, granularity-aligned): backed by the rank's own physical
// memory, or (ring >= 0) a mapping of broadcast-ring slot `ring` (a physical allocation of exactly
// len doubles, mapped at every block column that uses it).
struct VRegion { long long off, len; long long ring; };
struct VmmArena {
  CUdeviceptr base = 0;
  size_t size = 0;
  std::vector<std::pair<CUdeviceptr, size_t>> maps;
  std::vector<CUmemGenericAllocationHandle> phys;
  size_t phys_bytes = 0;
};
// Distributed top solve step: one outer block column [c0, c1) of top supernode J (the whole of J
// if it is not distributed), solved on its owner rank o.
struct TStep {
  int J, c0, c1, o;
  long long f0, f1, b0, b1;   // forward / backward tasks of the owner
};

}  // namespace spchol

struct spchol_handle {
  spchol::Symbolic S;
  spchol_options opt{};
  int nb = spchol::NBMAX;
  int outer = 4;                    // outer block = outer inner blocks (SPCHOL_OUTER, diagnostics)
  cudaStream_t stream = nullptr, own_stream = nullptr;
  // host plan
  std::vector<spchol::SnInfo> sn;
  std::vector<spchol::Launch> plan;
  std::vector<spchol::GTask> gtasks;
  std::vector<spchol::RTask> rtasks;    // RLB block-pair tiles (update_mode 1)
  std::vector<spchol::PTask> ptasks;
  std::vector<spchol::PanTask> pantasks;   // fused outer-block cdiv tiles (K_PANEL launches; aux = ticket index)
  int npanflags = 0, npanlaunch = 0;       // ready flags (16 per outer block) and K_PANEL launches
  bool panel_mode = true;                  // SPCHOL_PANEL=0: the cdiv as separate POTRF / TRSM / update launches
  int panel_grid = 0;                      // SPCHOL_PANEL_GRID: CTAs of a below launch (0 = min(tasks, 4 x 148))
  int panel_max_sn = 2;                    // SPCHOL_PANEL_MAX_SN: fused cdiv in levels with <= this many large supernodes
  int panel_max_rows = 6144;               // SPCHOL_PANEL_MAX_ROWS: ... for outer blocks with m - c0 <= this many rows
  std::vector<int> level_sns, level_off;
  std::vector<int> small_sns;           // supernodes handled by the fused small kernel, by level
  std::vector<char> is_small;
  long long panel_doubles = 0;          // panel arena (multi-GPU: the virtual extent of all ranks' panels)
  size_t device_bytes = 0;              // device memory the handle owns (SPCHOL_Q_DEVICE_BYTES)
  std::vector<long long> panel_off;
  std::vector<double> work;             // executed flops per supernode
  double flops_exec = 0, update_entries = 0;
  int nslots_total = 0;
  std::vector<int> slot_base;          // first inverse slot of each supernode's diagonal blocks
  // ---- multi-GPU (dist.cu): proportional subtree-to-GPU mapping; phase A = own
  // subtrees, exchange of the boundary blocks, phase C = top levels (distributed cdiv with
  // block-column broadcasts, partial U_J exchanged after each level)
  int rank = 0, world = 1;
  std::vector<int> owner;              // rank owning each supernode's subtree, -1 = top
  std::vector<int> top_owner;          // rank factoring each undistributed top supernode (LPT per level)
  std::vector<int> grp_lo, grp_hi;     // rank group [lo, hi) of each top supernode
  std::vector<char> top_dist;          // top supernode distributed over its group (block-column cyclic)
  double dist_min_flops = 4e9;         // SPCHOL_DIST_MINFLOPS: smallest top supernode distributed
  std::vector<size_t> markers;         // plan positions of the phase-C markers (same sequence on all ranks)
  std::vector<std::vector<int>> top_by_level;
  size_t plan_all_end = 0, plan_a_end = 0, plan_factor_begin = 0;
  int nvr = 1;                         // single-GPU subtree concurrency (virtual ranks)
  void* nccl_comm = nullptr;
  std::vector<std::array<int, 2>> grp_keys;   // distinct rank groups [lo, hi) of the top supernodes (hi - lo < world)
  std::vector<void*> grp_comms;               // their NCCL communicators (ncclCommSplit; null if not a member)
  // arena layout (multi-GPU): subtree region of each rank, own / aliased regions of this rank
  std::vector<long long> sub_off;      // [world + 1]
  std::vector<spchol::VRegion> vregions;
  long long ring_bytes = 0;            // this rank's broadcast ring (non-owned block columns map its slots)
  std::vector<long long> ring_slot_len; // doubles per ring slot
  std::vector<int> slot_sub;           // [world + 1] inverse-slot range of each rank's subtrees; top slots after
  // update blocks and the exchange
  std::vector<spchol::XBlk> xblk;
  std::vector<spchol::XRun> xrun;
  int nexch = 0;
  std::vector<std::vector<int>> exch_runs;   // per exchange: run indices, global order
  long long upd_off = 0, upd_doubles = 0, recv_off = 0, recv_doubles = 0;
  std::vector<spchol::XTask> xtasks;   // extend-add tasks of this rank, per exchange [xt_off[e], xt_off[e+1])
  std::vector<long long> xt_off, xcol;
  std::vector<int> xpos;
  double comm_send = 0, comm_recv = 0; // bytes per factor, this rank (exchanges + broadcasts)
  double comm_b_send = 0, comm_b_recv = 0;   // ... of the boundary-block exchange after phase A
  int ring_ns = 3;                     // ring slots per distributed top supernode
  // distributed solve
  std::vector<spchol::TStep> tsteps;
  std::vector<unsigned char> row_mine; // final row -> this rank holds its solution component
  // device (multi-GPU)
  spchol::VmmArena va_panels, va_linv;
  std::vector<CUmemGenericAllocationHandle> ring_phys;
  spchol::XTask* d_xtasks = nullptr;
  long long* d_xcol = nullptr;
  int* d_xpos = nullptr;
  unsigned char* d_row_mine = nullptr;
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_comm_in = nullptr, ev_comm_out = nullptr;
  bool graph_dist = false;             // the multi-GPU factor runs as a captured graph (real NCCL)
  bool dist_eager_done = false, dist_solve_eager_done = false, dist_capture_failed = false;
  // memory-capped mode (f-4, single GPU): resident top + subtree batches sharing one device window
  bool capped = false;
  std::vector<int> batch;                // batch of each supernode, -1 = resident top
  int nbatch = 0;
  std::vector<long long> batch_len;      // doubles of each batch's panels (a prefix of the window)
  std::vector<long long> batch_host;     // [nbatch + 1] offsets of the batches in the host copy
  std::vector<long long> host_off;       // per batch supernode: offset of its panel in the host copy
  long long window_doubles = 0, top_base = 0;
  std::vector<size_t> plan_batch;        // [nbatch + 1]: batch b's plan [plan_batch[b], plan_batch[b+1]); top after
  std::vector<long long> ainit_off;      // [nbatch + 2]: A's entries to initialise per batch, the top's last
  std::vector<long long> ainit_idx, ainit_dst;
  long long *d_ainit_idx = nullptr, *d_ainit_dst = nullptr;
  double* h_panels = nullptr;            // pinned host copy of the finished batches' panels
  struct SolveSeg { std::vector<long long> fwd, bwd; std::vector<int> ss; };
  std::vector<SolveSeg> segs;            // capped: per batch, then the top
  // single-GPU subtree concurrency etc.
  std::vector<int> small_level_off;     // small_sns range per level
  std::vector<spchol::STask> stasks;    // level solve tasks: forward of level l at [sfwd_off[l], sfwd_off[l+1]),
  std::vector<long long> sfwd_off, sbwd_off;   // backward at [sbwd_off[l], sbwd_off[l+1])
  spchol::STask* d_stasks = nullptr;
  std::vector<spchol::SmallSolve> ssolve;   // small supernodes, per level by row class (m <= 64 / 128 / 256)
  std::vector<int> ssolve_off;          // level l, class c at [ssolve_off[3l + c], ssolve_off[3l + c + 1])
  spchol::SmallSolve* d_ssolve = nullptr;
  int* d_sflags = nullptr;              // forward flags | backward flags | backward chunk counts (nslots
                                        // each) | tickets (2 per level and 2 per top step); zeroed per solve
  size_t nticket = 0;
  int nevents = 0;
  bool no_lookahead = false;     // SPCHOL_NO_LOOKAHEAD=1 (diagnostics)
  bool no_next_split = false;    // SPCHOL_NO_NEXT_SPLIT=1: NEXT as one critical-stream launch (diagnostics)
  int rest_smem = 0;             // SPCHOL_REST_SMEM: dynamic shared memory of trailing-stream updates (bytes)
  int left_inner_min = 16;       // SPCHOL_LEFT_INNER_MIN=n: left-looking in-block updates in levels with at
                                 // least n large supernodes (0 = never); SPCHOL_LEFT_INNER=1: everywhere
  bool right_inner = true;       // SPCHOL_LEFT_INNER=1: left-looking in-block updates (one K <= 192 pass
                                 // per block column; C4 -0.45%, C5 -0.35%, but C3/C2 +1.3-1.5%: on the chain)
  int max_level = -1;            // SPCHOL_MAX_LEVEL=l: factor only levels <= l (diagnostics)
  bool small_warp = true;        // SPCHOL_SMALL_WARP=0: CTA-per-supernode small kernel for every size
  int small_warp_maxm = 64;      // largest m of the warp-per-supernode kernel (SPCHOL_SMALL_WARP_MAXM <= 128)
  bool use_tma = false;          // SPCHOL_TMA=1: TMA + mbarrier tile kernels (measured ~2% slower)
  void* d_tmaps = nullptr;       // CUtensorMap per supernode panel (TMA boxes 16 x 8, 128B swizzle)
  void* d_tmap_linv = nullptr;   // CUtensorMap over the diagonal-inverse slots
  std::vector<int> plan_level;   // level of each plan entry (diagnostics)
  // device
  double *d_panels = nullptr, *d_avals = nullptr, *d_linv = nullptr, *d_y = nullptr, *d_y2 = nullptr;
  long long *d_diag_idx = nullptr, *d_amap = nullptr, *d_ucol_base = nullptr, *d_ucol_map = nullptr, *d_rows_ptr = nullptr;
  int *d_small_sns = nullptr, *d_posmap = nullptr, *d_sfirst = nullptr, *d_rows = nullptr, *d_perm = nullptr, *d_level_sns = nullptr;
  spchol::SnInfo* d_sn = nullptr;
  spchol::GTask* d_gtasks = nullptr;
  spchol::RTask* d_rtasks = nullptr;
  spchol::PTask* d_ptasks = nullptr;
  spchol::PanTask* d_pantasks = nullptr;
  int* d_pansync = nullptr;             // [npanflags] ready flags | 3 per K_PANEL launch (tickets, done count), zeroed per factor
  unsigned long long* d_fail = nullptr;
  bool values_set = false, factored = false;
  std::vector<cudaStream_t> pstreams;           // plan streams: even = cdiv chain (high priority),
                                                // odd = trailing updates (low priority)
  std::vector<cudaEvent_t> join_events;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  int prio_lo = 0, prio_hi = 0;
  std::vector<cudaEvent_t> plan_events;
  // graph
  cudaGraph_t graph = nullptr, solve_graph[3] = {nullptr, nullptr, nullptr};   // solve: per nr = 1, 2, 4
  cudaGraphExec_t gexec = nullptr, solve_gexec[3] = {nullptr, nullptr, nullptr};
  // spchol_set_values zeroes the arena on zstream while A's values travel (single GPU, resident): the
  // next factor then replays the variant graph without the memset
  bool prezeroed = false, skip_zero = false;
  cudaGraph_t graph_nz = nullptr;
  cudaGraphExec_t gexec_nz = nullptr;
  cudaStream_t zstream = nullptr;
  cudaEvent_t ev_zs = nullptr, ev_zd = nullptr;
  // timing
  bool timing = false;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  std::vector<std::pair<int, size_t>> pending;  // (plan index, first event)
  long long st_launches[spchol::K_NKINDS] = {0};
  double st_ms[spchol::K_NKINDS] = {0}, st_flops[spchol::K_NKINDS] = {0}, st_bytes[spchol::K_NKINDS] = {0};
};

namespace spchol {
// Multi-GPU distributed top supernode J (top_dist): outer column block C (columns [C W, (C+1) W),
// W = outer * nb) belongs to rank grp_lo + (C + top_owner - grp_lo) mod g — cyclic over J's rank
// group, starting at the rank the per-level LPT picked; an undistributed top supernode belongs to
// top_owner.
inline int blk_owner(const spchol_handle* h, int J, int C) {
  if (!h->top_dist[J]) return h->top_owner[J];
  const int g = h->grp_hi[J] - h->grp_lo[J];
  return h->grp_lo[J] + (C + h->top_owner[J] - h->grp_lo[J]) % g;
}
inline bool in_group(const spchol_handle* h, int J, int r) { return r >= h->grp_lo[J] && r < h->grp_hi[J]; }
inline int outer_w(const spchol_handle* h) { return h->outer * h->nb; }
// Number of outer blocks of a top supernode's ownership (1 if it is not distributed).
inline int top_nblk(const spchol_handle* h, int J) {
  return h->top_dist[J] ? (h->sn[J].k + outer_w(h) - 1) / outer_w(h) : 1;
}
void* group_comm(const spchol_handle* h, int J);

// dist.cu
void dist_layout(spchol_handle* h);                      // arena / inverse-slot layout of every rank
void dist_exchange_plan(spchol_handle* h);               // update blocks, runs, exchanges, extend-add tasks
void dist_solve_plan(spchol_handle* h);                  // per-rank level lists + top steps
void dist_redirect(const spchol_handle* h, std::vector<int>& posmap, std::vector<long long>& ucb);
bool dist_amap_mine(const spchol_handle* h, int col);    // this rank initialises A's entries of column col
int dist_setup_device(spchol_handle* h);                 // VMM arenas, exchange metadata
void dist_free_device(spchol_handle* h);
int dist_enqueue_init(spchol_handle* h, cudaStream_t st);
int dist_enqueue_exchange(spchol_handle* h, cudaStream_t st, int e);
int dist_enqueue_bcast(spchol_handle* h, cudaStream_t st, int J, int C);
int dist_enqueue_solve(spchol_handle* h, double* d_y2, int nr, cudaStream_t st);
bool dist_owns(const spchol_handle* h, int J, int col);  // this rank holds column col of supernode J
}  // namespace spchol
