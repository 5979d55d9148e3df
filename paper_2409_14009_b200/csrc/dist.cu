// Multi-GPU factorization and solve (north_star "partitioned across the 8xB200 box by
// subtree-to-GPU mapping of the etree ... boundary update matrices travel with NCCL send/recv over
// NVLink to the GPU that owns the ancestor").  One process per GPU; every rank builds the same
// global map (csrc/mapping.cpp) and its own plan.
//
// Memory.  Every rank reserves one virtual range laid out identically on all ranks — each rank's
// subtree panels, then the top supernodes' panels (a distributed one with its leading dimension
// padded so every W-column block column is a whole number of 2 MB pages) — and backs with physical
// memory (CUDA virtual memory management) only what it holds: its own subtrees, the top supernodes
// it factors whole, the block columns it owns of the distributed ones, and its update / receive
// regions.  The block columns of a distributed supernode that another rank owns are aliases into a
// small ring (ring_ns slots per supernode): a broadcast block column lives there only while the
// trailing updates that read it run.  Kernels address every panel exactly as on one GPU.
//
// Data flow of one factor:
//   phase A   each rank factors its subtrees; every update a subtree sends above its root S lands
//             in S's boundary block B_S over R_S x R_S (containment), through the same fused
//             SYRK + relind scatter with redirected targets (dist_redirect);
//   exchange  B_S is cut into column runs by destination (ancestor P, block column C); each run is
//             one ncclSend to the owner of (P, C) (ncclRecv there), all in one NCCL group; the owner
//             extend-adds the runs it receives (and its own) into its panels (extend_add_kernel);
//   phase C   top levels in order: the cdiv of a distributed top supernode runs block column by
//             block column on the owners, each finished block column is broadcast to the group
//             (ncclBroadcast), every member applies the trailing updates to the block columns it
//             owns; each member's partial U_J (its own block columns' share of the K sum) goes to
//             its update block of J, exchanged after the level like the boundary blocks.
// Solve: subtrees locally; top supernodes block column by block column on the owner, with a reduce
// of the block's partial right-hand side before the forward step and a broadcast of the block's
// solution after the backward step (only solution segments travel); one all-reduce of the
// masked solution at the end.
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include <cudaTypedefs.h>

#include "handle.h"

namespace spchol {

namespace {
constexpr long long GRAN = 2LL << 20;          // VMM mapping granularity (bytes)
constexpr long long GD = GRAN / 8;             // ... in doubles
constexpr int GS = (int)(GRAN / (NBMAX * NBMAX * 8));   // inverse slots per granule (64)
long long al(long long x, long long a) { return (x + a - 1) / a * a; }

// ---------------------------------------------------------------------------- VMM (driver API)
struct Vmm {
  PFN_cuMemCreate_v10020 create = nullptr;
  PFN_cuMemRelease_v10020 release = nullptr;
  PFN_cuMemAddressReserve_v10020 reserve = nullptr;
  PFN_cuMemAddressFree_v10020 vfree = nullptr;
  PFN_cuMemMap_v10020 map = nullptr;
  PFN_cuMemUnmap_v10020 unmap = nullptr;
  PFN_cuMemSetAccess_v10020 access = nullptr;
  PFN_cuMemGetAllocationGranularity_v10020 gran = nullptr;
  bool ok = false;
};
Vmm g_vmm;
int vmm_load() {
  if (g_vmm.ok) return SPCHOL_OK;
  cudaDriverEntryPointQueryResult q;
  auto get = [&](const char* nm, void** f) {
    return cudaGetDriverEntryPoint(nm, f, cudaEnableDefault, &q) == cudaSuccess && *f && q == cudaDriverEntryPointSuccess;
  };
  Vmm v;
  if (!get("cuMemCreate", (void**)&v.create) || !get("cuMemRelease", (void**)&v.release) ||
      !get("cuMemAddressReserve", (void**)&v.reserve) || !get("cuMemAddressFree", (void**)&v.vfree) ||
      !get("cuMemMap", (void**)&v.map) || !get("cuMemUnmap", (void**)&v.unmap) ||
      !get("cuMemSetAccess", (void**)&v.access) || !get("cuMemGetAllocationGranularity", (void**)&v.gran))
    return fail(SPCHOL_ERR_CUDA, "CUDA virtual memory management entry points unavailable");
  v.ok = true;
  g_vmm = v;
  return SPCHOL_OK;
}
CUmemAllocationProp vmm_prop(int dev) {
  CUmemAllocationProp p;
  std::memset(&p, 0, sizeof(p));
  p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  p.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  p.location.id = dev;
  return p;
}
int cu_fail(CUresult r, const char* where) {
  return fail(r == CUDA_ERROR_OUT_OF_MEMORY ? SPCHOL_ERR_DEVICE_OOM : SPCHOL_ERR_CUDA,
              std::string(where) + " failed (CUresult " + std::to_string((int)r) + ")");
}
#define CU(call)                                   \
  do {                                             \
    CUresult r_ = (call);                          \
    if (r_ != CUDA_SUCCESS) return cu_fail(r_, #call); \
  } while (0)
int vmm_phys(int dev, size_t bytes, CUmemGenericAllocationHandle* hd) {
  const CUmemAllocationProp p = vmm_prop(dev);
  CU(g_vmm.create(hd, bytes, &p, 0));
  return SPCHOL_OK;
}
int vmm_map(VmmArena& A, int dev, size_t off, size_t bytes, CUmemGenericAllocationHandle hd, size_t hoff) {
  CU(g_vmm.map(A.base + off, bytes, hoff, hd, 0));
  A.maps.push_back({A.base + off, bytes});
  CUmemAccessDesc d;
  std::memset(&d, 0, sizeof(d));
  d.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  d.location.id = dev;
  d.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CU(g_vmm.access(A.base + off, bytes, &d, 1));
  return SPCHOL_OK;
}
// Reserve `bytes` of virtual address space and back the own regions (ring < 0) with one physical
// allocation each; ring regions map a whole ring slot (cuMemMap maps from offset 0 of an allocation).
int vmm_build(VmmArena& A, int dev, size_t bytes, const std::vector<VRegion>& regs,
              const std::vector<CUmemGenericAllocationHandle>& ring) {
  A.size = (size_t)al((long long)bytes, GRAN);
  CU(g_vmm.reserve(&A.base, A.size, GRAN, 0, 0));
  for (const VRegion& r : regs) {
    const size_t off = (size_t)r.off * 8, len = (size_t)r.len * 8;
    if (len == 0) continue;
    if (r.ring >= 0) {
      int rc = vmm_map(A, dev, off, len, ring[r.ring], 0);
      if (rc) return rc;
      continue;
    }
    CUmemGenericAllocationHandle hd;
    int rc = vmm_phys(dev, len, &hd);
    if (rc) return rc;
    A.phys.push_back(hd);
    A.phys_bytes += len;
    if ((rc = vmm_map(A, dev, off, len, hd, 0))) return rc;
  }
  return SPCHOL_OK;
}
void vmm_free(VmmArena& A) {
  if (!g_vmm.ok) return;
  for (auto& m : A.maps) g_vmm.unmap(m.first, m.second);
  for (auto hd : A.phys) g_vmm.release(hd);
  if (A.base) g_vmm.vfree(A.base, A.size);
  A = VmmArena();
}
}  // namespace

// ------------------------------------------------------------------------------- ownership
bool dist_owns(const spchol_handle* h, int J, int col) {
  if (h->owner[J] >= 0) return h->owner[J] == h->rank;
  const int C = h->top_dist[J] ? (col - h->S.sfirst[J]) / outer_w(h) : 0;
  return blk_owner(h, J, C) == h->rank;
}
bool dist_amap_mine(const spchol_handle* h, int col) { return dist_owns(h, h->S.snode[col], col); }

// ------------------------------------------------------------------------------- layout
void dist_layout(spchol_handle* h) {
  const Symbolic& S = h->S;
  const int ns = S.nsuper, P = h->world, r = h->rank, W = outer_w(h), NB = h->nb;
  long long off = 0;
  h->sub_off.assign(P + 1, 0);
  for (int q = 0; q < P; ++q) {
    h->sub_off[q] = off;
    for (int J = 0; J < ns; ++J)
      if (h->owner[J] == q) {
        h->sn[J].off = off;
        off += (long long)h->sn[J].ld * h->sn[J].k;
      }
    off = al(off, GD);
  }
  h->sub_off[P] = off;
  for (int J = 0; J < ns; ++J) {
    if (h->owner[J] >= 0) continue;
    off = al(off, GD);
    SnInfo& I = h->sn[J];
    if (h->top_dist[J]) I.ld = (int)al(I.m, GD / W);   // every block column = whole 2 MB pages
    I.off = off;
    // a distributed supernode's range covers whole block columns (each one a ring-slot mapping)
    off += (long long)I.ld * (h->top_dist[J] ? (long long)top_nblk(h, J) * W : I.k);
  }
  h->panel_doubles = al(off, GD);
  // diagonal-inverse slots: each rank's subtree slots, then every top slot (mapped on all ranks)
  h->slot_base.assign(ns, 0);
  h->slot_sub.assign(P + 1, 0);
  int slot = 0;
  for (int q = 0; q <= P; ++q) {
    h->slot_sub[q] = slot;
    for (int J = 0; J < ns; ++J) {
      if (h->is_small[J] || (q < P ? h->owner[J] != q : h->owner[J] >= 0)) continue;
      h->slot_base[J] = slot;
      slot += (h->sn[J].k + NB - 1) / NB;
    }
    slot = (int)al(slot, GS);
  }
  h->nslots_total = slot;
  // this rank's regions of the panel range: own physical memory, or ring aliases
  h->vregions.clear();
  if (h->sub_off[r + 1] > h->sub_off[r]) h->vregions.push_back({h->sub_off[r], h->sub_off[r + 1] - h->sub_off[r], -1});
  h->ring_slot_len.clear();
  h->ring_bytes = 0;
  for (int J = 0; J < ns; ++J) {
    if (h->owner[J] >= 0) continue;
    const SnInfo& I = h->sn[J];
    if (!h->top_dist[J]) {
      if (h->top_owner[J] == r) h->vregions.push_back({I.off, al((long long)I.ld * I.k, GD), -1});
      continue;
    }
    if (!in_group(h, J, r)) continue;
    const long long blk = (long long)I.ld * W;   // doubles per full block column (multiple of GD)
    long long ring0 = -1;                        // this supernode's ring_ns slots (C mod ring_ns)
    for (int C = 0; C * W < I.k; ++C) {
      if (blk_owner(h, J, C) == r) {
        h->vregions.push_back({I.off + (long long)C * blk, al((long long)I.ld * std::min(W, I.k - C * W), GD), -1});
      } else {
        if (ring0 < 0) {
          ring0 = (long long)h->ring_slot_len.size();
          for (int q = 0; q < h->ring_ns; ++q) h->ring_slot_len.push_back(blk);
          h->ring_bytes += 8LL * h->ring_ns * blk;
        }
        h->vregions.push_back({I.off + (long long)C * blk, blk, ring0 + C % h->ring_ns});
      }
    }
  }
}

// ------------------------------------------------------------------------------- exchange plan
namespace {
inline const int32_t* xrows(const spchol_handle* h, const XBlk& B) {
  return h->S.rows.data() + h->S.rows_ptr[B.node] + h->sn[B.node].k;
}
}  // namespace

void dist_exchange_plan(spchol_handle* h) {
  const Symbolic& S = h->S;
  const int ns = S.nsuper, P = h->world, r = h->rank, W = outer_w(h);
  h->xblk.clear();
  h->xrun.clear();
  h->nexch = 1 + S.nlevels;
  h->exch_runs.assign(h->nexch, {});
  auto add_block = [&](int src, int node, int exch, int kind) {
    const SnInfo& I = h->sn[node];
    const int t = I.m - I.k;
    if (t <= 0) return;
    XBlk B{src, node, exch, kind, t, (long long)h->xrun.size(), 0};
    const int32_t* R = S.rows.data() + S.rows_ptr[node] + I.k;
    int j0 = 0;
    while (j0 < t) {
      const int Pn = S.snode[R[j0]];
      const int C = h->top_dist[Pn] ? (R[j0] - S.sfirst[Pn]) / W : 0;
      const int cend = h->top_dist[Pn] ? std::min(S.sfirst[Pn] + (C + 1) * W, S.sfirst[Pn + 1]) : S.sfirst[Pn + 1];
      int j1 = j0 + 1;
      while (j1 < t && R[j1] < cend) ++j1;   // rows of R are sorted: the run ends at the block's end
      XRun X{(int)h->xblk.size(), j0, j1, Pn, C, blk_owner(h, Pn, C), 0, 0, 0};
      X.ld = (t - j0) + ((t - j0) & 1);
      h->xrun.push_back(X);
      j0 = j1;
    }
    B.run1 = (long long)h->xrun.size();
    h->xblk.push_back(B);
  };
  // boundary blocks: subtree roots whose parent is a top supernode (exchange 0, after phase A)
  for (int J = 0; J < ns; ++J)
    if (h->owner[J] >= 0 && S.sparent[J] >= 0 && h->owner[S.sparent[J]] < 0) add_block(h->owner[J], J, 0, 0);
  // partial U_J of the top supernodes: one per rank holding a block column (exchange 1 + level)
  for (int J = 0; J < ns; ++J) {
    if (h->owner[J] >= 0) continue;
    std::vector<int> holders;
    for (int C = 0; C < top_nblk(h, J); ++C) holders.push_back(blk_owner(h, J, C));
    std::sort(holders.begin(), holders.end());
    holders.erase(std::unique(holders.begin(), holders.end()), holders.end());
    for (int q : holders) add_block(q, J, 1 + S.level[J], 1);
  }
  // storage: per (source rank, exchange) consecutive runs in the update region; per (destination,
  // exchange) consecutive receives in the receive region (global order on every rank)
  std::vector<long long> uo(P, 0), ro(P, 0);
  std::vector<long long> umax(P, 0), rmax(P, 0);
  for (int e = 0; e < h->nexch; ++e) {
    std::fill(uo.begin(), uo.end(), 0);
    std::fill(ro.begin(), ro.end(), 0);
    for (size_t b = 0; b < h->xblk.size(); ++b) {
      const XBlk& B = h->xblk[b];
      if (B.exch != e) continue;
      for (long long x = B.run0; x < B.run1; ++x) {
        XRun& X = h->xrun[x];
        const long long sz = (long long)X.ld * (X.j1 - X.j0);
        X.loc = uo[B.src];
        uo[B.src] += sz;
        if (X.dst != B.src) {
          X.roff = ro[X.dst];
          ro[X.dst] += sz;
        }
        h->exch_runs[e].push_back((int)x);
      }
    }
    for (int q = 0; q < P; ++q) { umax[q] = std::max(umax[q], uo[q]); rmax[q] = std::max(rmax[q], ro[q]); }
  }
  h->upd_off = h->panel_doubles;
  h->upd_doubles = al(umax[r], GD);
  h->recv_off = h->upd_off + h->upd_doubles;
  h->recv_doubles = al(rmax[r], GD);
  if (h->upd_doubles) h->vregions.push_back({h->upd_off, h->upd_doubles, -1});
  if (h->recv_doubles) h->vregions.push_back({h->recv_off, h->recv_doubles, -1});
  // communication volume of this rank per factor (exchanges + broadcasts)
  h->comm_send = h->comm_recv = h->comm_b_send = h->comm_b_recv = 0;
  for (const XRun& X : h->xrun) {
    const double by = 8.0 * X.ld * (X.j1 - X.j0);
    const XBlk& B = h->xblk[X.blk];
    if (B.src == X.dst) continue;
    if (B.src == r) { h->comm_send += by; if (B.exch == 0) h->comm_b_send += by; }
    if (X.dst == r) { h->comm_recv += by; if (B.exch == 0) h->comm_b_recv += by; }
  }
  for (int J = 0; J < ns; ++J) {
    if (!h->top_dist[J] || !in_group(h, J, r)) continue;
    const SnInfo& I = h->sn[J];
    for (int C = 0; C * W < I.k; ++C) {
      const double by = 8.0 * I.ld * std::min(W, I.k - C * W);
      // logical volume: a broadcast counts once per receiving member on the owner's side
      if (blk_owner(h, J, C) == r) h->comm_send += by * (h->grp_hi[J] - h->grp_lo[J] - 1); else h->comm_recv += by;
    }
  }
  // extend-add tasks of this rank: every run it owns the destination of (received or its own)
  h->xtasks.clear();
  h->xcol.clear();
  h->xpos.clear();
  h->xt_off.assign(h->nexch + 1, 0);
  std::vector<int> pos(S.n, -1);
  int posP = -1;
  for (int e = 0; e < h->nexch; ++e) {
    h->xt_off[e] = (long long)h->xtasks.size();
    for (int x : h->exch_runs[e]) {
      const XRun& X = h->xrun[x];
      if (X.dst != r) continue;
      const XBlk& B = h->xblk[X.blk];
      const int32_t* R = xrows(h, B);
      const SnInfo& IP = h->sn[X.P];
      if (posP != X.P) {
        if (posP >= 0)
          for (long long q = S.rows_ptr[posP]; q < S.rows_ptr[posP + 1]; ++q) pos[S.rows[q]] = -1;
        for (long long q = S.rows_ptr[X.P]; q < S.rows_ptr[X.P + 1]; ++q) pos[S.rows[q]] = (int)(q - S.rows_ptr[X.P]);
        posP = X.P;
      }
      const long long cb = (long long)h->xcol.size(), pb = (long long)h->xpos.size();
      for (int j = X.j0; j < X.j1; ++j) h->xcol.push_back(IP.off + (long long)(R[j] - S.sfirst[X.P]) * IP.ld);
      for (int i = X.j0; i < B.t; ++i) h->xpos.push_back(pos[R[i]]);   // R[i] in rows(P): containment
      const long long src = B.src == r ? h->upd_off + X.loc : h->recv_off + X.roff;
      for (int c0 = 0; c0 < X.j1 - X.j0; c0 += 8)
        h->xtasks.push_back(XTask{src, cb, pb, X.ld, B.t - X.j0, c0, std::min(8, X.j1 - X.j0 - c0)});
    }
  }
  h->xt_off[h->nexch] = (long long)h->xtasks.size();
}

// Scatter targets of this rank's supernodes whose updates leave the rank: a subtree supernode D's
// pairs (D, P) with P top go to the boundary block of D's subtree root S (row = position in R_S);
// a top supernode J's pairs go to this rank's update block of J (row = position in R_J).  The U
// column c of D lands in the run holding it: ucol_base = run start + (j - j0) ld - j0, so that
// ucol_base + posmap = run start + (j - j0) ld + (i - j0) for U entry (row i, column j) of R.
void dist_redirect(const spchol_handle* h, std::vector<int>& posmap, std::vector<long long>& ucb) {
  const Symbolic& S = h->S;
  const int ns = S.nsuper, r = h->rank;
  std::vector<int> blk_of(ns, -1);   // update block of this rank for node (boundary block / partial U)
  for (size_t b = 0; b < h->xblk.size(); ++b)
    if (h->xblk[b].src == r) blk_of[h->xblk[b].node] = (int)b;
  std::vector<int> sroot(ns, -1);
  for (int J = ns - 1; J >= 0; --J) {
    if (h->owner[J] < 0) continue;
    const int p = S.sparent[J];
    sroot[J] = (p < 0 || h->owner[p] < 0) ? J : sroot[p];
  }
  std::vector<int> posX(S.n, -1);
  int cur = -1;
  auto fill = [&](int X) {   // posX[row] = index of row in R_X
    if (cur == X) return;
    if (cur >= 0)
      for (long long q = S.rows_ptr[cur]; q < S.rows_ptr[cur + 1]; ++q) posX[S.rows[q]] = -1;
    const int k = h->sn[X].k;
    for (long long q = S.rows_ptr[X] + k; q < S.rows_ptr[X + 1]; ++q) posX[S.rows[q]] = (int)(q - S.rows_ptr[X] - k);
    cur = X;
  };
  for (int D = 0; D < ns; ++D) {
    int X = -1;
    if (h->owner[D] == r && sroot[D] >= 0 && blk_of[sroot[D]] >= 0 && h->xblk[blk_of[sroot[D]]].kind == 0) X = sroot[D];
    else if (h->owner[D] < 0 && blk_of[D] >= 0) X = D;
    if (X < 0) continue;
    const SnInfo& I = h->sn[D];
    if (I.m <= I.k) continue;
    fill(X);
    const XBlk& B = h->xblk[blk_of[X]];
    const int32_t* rD = S.rows.data() + S.rows_ptr[D];
    for (long long p = S.rel_ptr[D]; p < S.rel_ptr[D + 1]; ++p) {
      if (h->owner[S.rel_anc[p]] >= 0) continue;   // ancestor inside the subtree: unchanged
      for (long long x = S.rel_off[p]; x < S.rel_off[p + 1]; ++x) posmap[x] = posX[rD[S.rel_q0[p] + (x - S.rel_off[p])]];
    }
    long long run = B.run0;
    for (int q = I.k; q < I.m; ++q) {
      if (h->owner[S.snode[rD[q]]] >= 0) continue;
      const int j = posX[rD[q]];
      while (h->xrun[run].j1 <= j) ++run;   // columns ascend with q
      const XRun& R = h->xrun[run];
      ucb[I.ucol + (q - I.k)] = h->upd_off + R.loc + (long long)(j - R.j0) * R.ld - R.j0;
    }
  }
}

// ------------------------------------------------------------------------------- solve plan
void dist_solve_plan(spchol_handle* h) {
  const Symbolic& S = h->S;
  const int ns = S.nsuper, NB = h->nb, W = outer_w(h);
  h->tsteps.clear();
  // top steps in forward order: levels ascending, supernodes ascending, block columns ascending
  for (int l = 0; l < S.nlevels; ++l)
    for (int x = h->level_off[l]; x < h->level_off[l + 1]; ++x) {
      const int J = h->level_sns[x];
      if (h->owner[J] >= 0 || h->sn[J].k == 0) continue;
      const SnInfo& I = h->sn[J];
      for (int C = 0; C < top_nblk(h, J); ++C) {
        const int c0 = h->top_dist[J] ? C * W : 0, c1 = h->top_dist[J] ? std::min(I.k, c0 + W) : I.k;
        TStep T{J, c0, c1, blk_owner(h, J, C), 0, 0, 0, 0};
        h->tsteps.push_back(T);
      }
    }
  // tasks of the steps this rank owns (the solve's level kernels with bounded column blocks)
  for (TStep& T : h->tsteps) {
    T.f0 = T.f1 = T.b0 = T.b1 = (long long)h->stasks.size();
    if (T.o != h->rank) continue;
    const SnInfo& I = h->sn[T.J];
    const int J = T.J;
    const int cb0 = T.c0 / NB, cb1 = (T.c1 + NB - 1) / NB;
    for (int b = cb0; b < cb1; ++b) {
      const int nb = std::min(NB, I.k - b * NB);
      h->stasks.push_back(STask{J, 0, b, nb, b * NB, b * NB + nb, h->slot_base[J] + b, 0, cb0, cb1});
    }
    for (int q0 = T.c1; q0 < I.m; q0 += 64)
      h->stasks.push_back(STask{J, 1, 0, 0, q0, std::min(q0 + 64, I.m), h->slot_base[J], 0, cb0, cb1});
    T.f1 = T.b0 = (long long)h->stasks.size();
    const int need = (I.m - T.c1 + SOLVE_RCHUNK - 1) / SOLVE_RCHUNK;
    for (int b = cb0; b < cb1; ++b)
      for (int q0 = T.c1; q0 < I.m; q0 += SOLVE_RCHUNK)
        h->stasks.push_back(STask{J, 2, b, std::min(NB, I.k - b * NB), q0, std::min(q0 + SOLVE_RCHUNK, I.m),
                                  h->slot_base[J] + b, 0, cb0, cb1});
    for (int b = cb1 - 1; b >= cb0; --b) {
      const int nb = std::min(NB, I.k - b * NB);
      h->stasks.push_back(STask{J, 3, b, nb, b * NB, b * NB + nb, h->slot_base[J] + b, need, cb0, cb1});
    }
    T.b1 = (long long)h->stasks.size();
  }
  h->nticket = 2 * ((size_t)S.nlevels + h->tsteps.size());
  // the rank holding each solution component at the end (subtree rows: their owner; top rows: the
  // owner of their block column)
  h->row_mine.assign(S.n, 0);
  for (int J = 0; J < ns; ++J)
    for (int c = S.sfirst[J]; c < S.sfirst[J + 1]; ++c) h->row_mine[c] = dist_owns(h, J, c) ? 1 : 0;
}

// ------------------------------------------------------------------------------- device
int dist_setup_device(spchol_handle* h) {
  int rc = vmm_load();
  if (rc) return rc;
  const int dev = h->opt.device;
  size_t gmin = 0;
  {
    const CUmemAllocationProp p = vmm_prop(dev);
    CU(g_vmm.gran(&gmin, &p, CU_MEM_ALLOC_GRANULARITY_MINIMUM));
    if (gmin == 0 || GRAN % (long long)gmin != 0) return fail(SPCHOL_ERR_CUDA, "unsupported VMM granularity");
  }
  for (long long len : h->ring_slot_len) {
    h->ring_phys.push_back(0);
    if ((rc = vmm_phys(dev, (size_t)len * 8, &h->ring_phys.back()))) return rc;
  }
  if ((rc = vmm_build(h->va_panels, dev, (size_t)(h->recv_off + h->recv_doubles) * 8, h->vregions, h->ring_phys))) return rc;
  h->d_panels = (double*)h->va_panels.base;
  // inverse slots: own subtree range + every top slot
  std::vector<VRegion> lr;
  const long long SL = (long long)NBMAX * NBMAX;
  const int r = h->rank, P = h->world;
  if (h->slot_sub[r + 1] > h->slot_sub[r]) lr.push_back({h->slot_sub[r] * SL, (h->slot_sub[r + 1] - h->slot_sub[r]) * SL, -1});
  if (h->nslots_total > h->slot_sub[P]) lr.push_back({h->slot_sub[P] * SL, (h->nslots_total - h->slot_sub[P]) * SL, -1});
  if ((rc = vmm_build(h->va_linv, dev, (size_t)std::max(1, h->nslots_total) * SL * 8, lr, {}))) return rc;
  h->d_linv = (double*)h->va_linv.base;
  g_dev_bytes += h->va_panels.phys_bytes + h->va_linv.phys_bytes + (size_t)h->ring_bytes;
  CK(upload(&h->d_xtasks, h->xtasks));
  CK(upload(&h->d_xcol, h->xcol));
  CK(upload(&h->d_xpos, h->xpos));
  CK(upload(&h->d_row_mine, h->row_mine));
  int lo = 0, hi = 0;
  CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  CK(cudaStreamCreateWithPriority(&h->comm_stream, cudaStreamNonBlocking, hi));
  CK(cudaEventCreateWithFlags(&h->ev_comm_in, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&h->ev_comm_out, cudaEventDisableTiming));
  return SPCHOL_OK;
}

void dist_free_device(spchol_handle* h) {
  void* ptrs[] = {h->d_xtasks, h->d_xcol, h->d_xpos, h->d_row_mine};
  for (void* p : ptrs) if (p) cudaFree(p);
  if (h->ev_comm_in) cudaEventDestroy(h->ev_comm_in);
  if (h->ev_comm_out) cudaEventDestroy(h->ev_comm_out);
  if (h->comm_stream) cudaStreamDestroy(h->comm_stream);
  if (h->d_panels || h->d_linv) cudaDeviceSynchronize();
  vmm_free(h->va_panels);
  vmm_free(h->va_linv);
  if (g_vmm.ok) for (auto hd : h->ring_phys) if (hd) g_vmm.release(hd);
  h->ring_phys.clear();
  h->d_panels = nullptr;
  h->d_linv = nullptr;
}

// a1 under multi-GPU: zero what this rank holds (own physical regions, incl. the update region),
// then A's entries of the columns it owns.
int dist_enqueue_init(spchol_handle* h, cudaStream_t st) {
  CK(cudaMemsetAsync(h->d_fail, 0xFF, sizeof(unsigned long long), st));
  for (const VRegion& g : h->vregions)
    if (g.ring < 0 && g.off < h->recv_off) CK(cudaMemsetAsync(h->d_panels + g.off, 0, sizeof(double) * (size_t)g.len, st));
  launch_init(h->d_avals, h->d_amap, h->S.nnzA, h->d_panels, st);
  CK(cudaGetLastError());
  return SPCHOL_OK;
}

// Exchange e: after the work on stream st (phase A, or a top level) the update runs travel to the
// owners of their destination block columns (one NCCL group of sends and receives on the comm
// stream), are extend-added there, and the update region is zeroed for the next producer; st then
// waits for all of it.
int dist_enqueue_exchange(spchol_handle* h, cudaStream_t st, int e) {
  if (!h->nccl_comm) return fail(SPCHOL_ERR_STATE, "multi-GPU handle without an NCCL communicator (spchol_dist_attach_nccl)");
  cudaStream_t cs = h->comm_stream;
  CK(cudaEventRecord(h->ev_comm_in, st));
  CK(cudaStreamWaitEvent(cs, h->ev_comm_in, 0));
  const int r = h->rank;
  int rc = g_nccl.group_start();
  if (rc) return nccl_fail(rc, "ncclGroupStart");
  for (int x : h->exch_runs[e]) {
    const XRun& X = h->xrun[x];
    const int src = h->xblk[X.blk].src;
    if (src == X.dst) continue;
    const size_t cnt = (size_t)X.ld * (X.j1 - X.j0);
    if (src == r) rc = g_nccl.send(h->d_panels + h->upd_off + X.loc, cnt, NCCL_FLOAT64, X.dst, h->nccl_comm, cs);
    else if (X.dst == r) rc = g_nccl.recv(h->d_panels + h->recv_off + X.roff, cnt, NCCL_FLOAT64, src, h->nccl_comm, cs);
    if (rc) { g_nccl.group_end(); return nccl_fail(rc, "ncclSend/ncclRecv(update run)"); }
  }
  rc = g_nccl.group_end();
  if (rc) return nccl_fail(rc, "ncclGroupEnd");
  launch_extend_add(h->d_xtasks + h->xt_off[e], (int)(h->xt_off[e + 1] - h->xt_off[e]), h->d_xcol, h->d_xpos, h->d_panels, cs);
  if (h->upd_doubles) CK(cudaMemsetAsync(h->d_panels + h->upd_off, 0, sizeof(double) * (size_t)h->upd_doubles, cs));
  CK(cudaEventRecord(h->ev_comm_out, cs));
  CK(cudaStreamWaitEvent(st, h->ev_comm_out, 0));
  CK(cudaGetLastError());
  return SPCHOL_OK;
}

// Block column C of distributed top supernode J is final on its owner: broadcast to J's rank group
// (ncclBroadcast on the group's communicator, into the members' ring aliases of that block column).
// The owner's stream does not wait for the broadcast (it only reads the block); the members' do.
int dist_enqueue_bcast(spchol_handle* h, cudaStream_t st, int J, int C) {
  if (!h->nccl_comm) return fail(SPCHOL_ERR_STATE, "multi-GPU handle without an NCCL communicator (spchol_dist_attach_nccl)");
  if (!in_group(h, J, h->rank)) return SPCHOL_OK;
  const int W = outer_w(h), o = blk_owner(h, J, C);
  const SnInfo& I = h->sn[J];
  const int c0 = C * W, nc = std::min(W, I.k - c0);
  double* p = h->d_panels + I.off + (size_t)c0 * I.ld;
  void* comm = group_comm(h, J);
  if (!comm) return fail(SPCHOL_ERR_STATE, "no communicator for a top rank group");
  cudaStream_t cs = h->comm_stream;
  CK(cudaEventRecord(h->ev_comm_in, st));
  CK(cudaStreamWaitEvent(cs, h->ev_comm_in, 0));
  const int rc = g_nccl.bcast(p, p, (size_t)I.ld * nc, NCCL_FLOAT64, o - h->grp_lo[J], comm, cs);
  if (rc) return nccl_fail(rc, "ncclBroadcast(block column)");
  CK(cudaEventRecord(h->ev_comm_out, cs));
  if (o != h->rank) CK(cudaStreamWaitEvent(st, h->ev_comm_out, 0));
  return SPCHOL_OK;
}

// Distributed solve of the permuted system in place on d_y2 (original numbering in and out).
int dist_enqueue_solve(spchol_handle* h, double* d_y2, int nr, cudaStream_t st) {
  if (!h->nccl_comm) return fail(SPCHOL_ERR_STATE, "multi-GPU handle without an NCCL communicator");
  const Symbolic& S = h->S;
  const size_t NS = (size_t)std::max(1, h->nslots_total);
  int* fflag = h->d_sflags;
  int* bflag = fflag + NS;
  int* rcnt = bflag + NS;
  int* tickets = rcnt + NS;
  CK(cudaMemsetAsync(h->d_sflags, 0, sizeof(int) * (3 * NS + h->nticket), st));
  launch_permute_masked(h->d_perm, h->d_row_mine, d_y2, h->d_y, S.n, nr, 0, st);   // b counted once: on its row's owner
  for (int l = 0; l < S.nlevels; ++l) {
    for (int cl = 0; cl < 3; ++cl)
      launch_solve_small(h->d_ssolve + h->ssolve_off[3 * l + cl], h->ssolve_off[3 * l + cl + 1] - h->ssolve_off[3 * l + cl],
                         cl, 0, h->d_rows, h->d_panels, h->d_y, nr, st);
    launch_solve_fwd_level(h->d_stasks + h->sfwd_off[l], (int)(h->sbwd_off[l] - h->sfwd_off[l]), tickets + 2 * l, fflag,
                           h->d_sn, h->d_sfirst, h->d_rows_ptr, h->d_rows, h->d_panels, h->d_linv, h->d_y, h->nb, nr, st);
  }
  int* tt = tickets + 2 * S.nlevels;
  for (size_t s = 0; s < h->tsteps.size(); ++s) {   // forward: the block's partial sums onto its owner
    const TStep& T = h->tsteps[s];
    if (!in_group(h, T.J, h->rank)) continue;
    double* yb = h->d_y + (size_t)(S.sfirst[T.J] + T.c0) * nr;
    const int rc = g_nccl.reduce(yb, yb, (size_t)(T.c1 - T.c0) * nr, NCCL_FLOAT64, NCCL_SUM, T.o - h->grp_lo[T.J], group_comm(h, T.J), st);
    if (rc) return nccl_fail(rc, "ncclReduce(solve block)");
    if (T.o == h->rank)
      launch_solve_fwd_level(h->d_stasks + T.f0, (int)(T.f1 - T.f0), tt + 2 * s, fflag, h->d_sn, h->d_sfirst, h->d_rows_ptr,
                             h->d_rows, h->d_panels, h->d_linv, h->d_y, h->nb, nr, st);
  }
  for (size_t s = h->tsteps.size(); s-- > 0;) {   // backward: the block's solution to the group
    const TStep& T = h->tsteps[s];
    if (!in_group(h, T.J, h->rank)) continue;
    if (T.o == h->rank)
      launch_solve_bwd_level(h->d_stasks + T.b0, (int)(T.b1 - T.b0), tt + 2 * s + 1, bflag, rcnt, h->d_sn, h->d_sfirst,
                             h->d_rows_ptr, h->d_rows, h->d_panels, h->d_linv, h->d_y, h->nb, nr, st);
    double* yb = h->d_y + (size_t)(S.sfirst[T.J] + T.c0) * nr;
    const int rc = g_nccl.bcast(yb, yb, (size_t)(T.c1 - T.c0) * nr, NCCL_FLOAT64, T.o - h->grp_lo[T.J], group_comm(h, T.J), st);
    if (rc) return nccl_fail(rc, "ncclBroadcast(solve block)");
  }
  for (int l = S.nlevels - 1; l >= 0; --l) {
    launch_solve_bwd_level(h->d_stasks + h->sbwd_off[l], (int)(h->sfwd_off[l + 1] - h->sbwd_off[l]), tickets + 2 * l + 1,
                           bflag, rcnt, h->d_sn, h->d_sfirst, h->d_rows_ptr, h->d_rows, h->d_panels, h->d_linv, h->d_y,
                           h->nb, nr, st);
    for (int cl = 0; cl < 3; ++cl)
      launch_solve_small(h->d_ssolve + h->ssolve_off[3 * l + cl], h->ssolve_off[3 * l + cl + 1] - h->ssolve_off[3 * l + cl],
                         cl, 1, h->d_rows, h->d_panels, h->d_y, nr, st);
  }
  launch_permute_masked(h->d_perm, h->d_row_mine, h->d_y, d_y2, S.n, nr, 1, st);   // each component from its holder
  const int rc = g_nccl.allreduce(d_y2, d_y2, (size_t)S.n * nr, NCCL_FLOAT64, NCCL_SUM, h->nccl_comm, st);
  if (rc) return nccl_fail(rc, "ncclAllReduce(solution)");
  CK(cudaGetLastError());
  return SPCHOL_OK;
}

}  // namespace spchol
