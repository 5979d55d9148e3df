// sm_100a device kernels of the numeric RL factorization (arXiv 2409.14009, §II.A "RL").
// P:n = PAPER.md line n.  All arithmetic is FP64 ("D" BLAS).
//
//   potrf10_kernel      a3: cdiv POTRF of one <=64-column diagonal block in shared memory, plus its
//                       triangular inverse (used by TRSM-as-GEMM and the solve)  ("DPOTRF");
//                       potrf9_kernel: the right-looking reference (SPCHOL_POTRF9=1)
//   gemm_kernel<MODE>   FP64 DMMA (mma.sync m8n8k4) 64x64 tile, cp.async 4-stage smem pipeline
//     MODE_TRSM         a4: L_{R,b} = A_{R,b} L_bb^{-T}                          ("DTRSM")
//     MODE_LOCAL        right-looking update of the supernode's own trailing columns
//     MODE_SCATTER      a5+a6: U_J = L_{R,J} L_{R,J}^T ("DSYRK") with the relind assembly
//                        fused into the epilogue: FP64 RED into ancestors
//   panel_diag_kernel / panel_below_kernel
//                       a3+a4 fused: the cdiv of one 256-column outer block (its lookahead update by
//                       the previous outer block, POTRF, TRSM and the in-block updates of every 64-row
//                       tile) in one launch pair, flag-synchronised
//   init_scatter        a1: A's entries into the zeroed panel arena
//   solve kernels       forward / backward supernodal triangular solves
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace spchol {

// Panel J: column-major m x k rectangle at panels + off, leading dimension ld (even, >= m).
struct SnInfo {
  long long off;
  int ld, m, k, ucol;  // ucol: first U-column descriptor of J (see MODE_SCATTER)
};
// A GEMM tile task; meaning of the fields per mode is documented in gemm_kernel.
struct GTask {
  int sn, r0, s0, c0, nb, slot;
};
struct PTask {
  int sn, c0, nb, slot;
};
// RLB tile task: the 64-row windows [ra, ra+64) x [rb, rb+64) of supernode sn's update
// (ra, rb even: 16-byte aligned loads) restricted to one block pair: window rows [i0, i1) of block
// B', columns [j0, j1) of block B.  Entry (i, j) goes to the ancestor panel at
// dst + (j - j0) * ldd + (i - i0); diag (B == B'): only ra + i >= rb + j.
struct RTask {
  int sn, ra, rb, i0, i1, j0, j1, diag;
  long long dst;
  int ldd, pad;
};
// Solve task of one level (sync-free blocked triangular solve, solve_fwd_level / solve_bwd_level).
// kind 0: forward, triangle row block cb (rows [q0, q1) = the block's columns);
// kind 1: forward, rows [q0, q1) >= k of the panel (all column blocks; RED into the ancestors);
// kind 2: backward, column block cb against rows [q0, q1) >= k (partial dot products, RED into y_cb);
// kind 3: backward, triangle column block cb (waits for `need` kind-2 chunks and the blocks > cb).
// slot = diagonal-inverse slot of block cb (slot - cb = slot of block 0 = the flag base).
// cblo / cbhi bound the column blocks a task sums over (single GPU: 0 / all blocks; the distributed
// top solve restricts them to one rank's outer block column): kind 0 sums cb in [cblo, cb), kind 1
// cb in [cblo, cbhi), kind 3 rb in (cb, cbhi).
struct STask {
  int sn, kind, cb, nb, q0, q1, slot, need, cblo, cbhi;
};
// MODE_SCATTER_DET: MODE_SCATTER with plain RMW stores (deterministic mode: the launch's supernodes are
// column-conflict free, so no two CTAs of the launch touch one ancestor entry).
// MODE_SCATTER_KS (multi-GPU, distributed top supernode): MODE_SCATTER over this rank's share of the
// K columns only — the owned outer block columns c0 + i * slot (i < nb), kw columns each — so the
// group's partial U_J sum to U_J (P:307 with the sum over the columns of L_J split by owner).
enum { MODE_LOCAL = 0, MODE_TRSM = 1, MODE_SCATTER = 2, MODE_RLB = 3, MODE_SCATTER_DET = 4, MODE_SCATTER_KS = 5 };
// Extend-add task (multi-GPU exchange): columns [c0, c0 + nc) of one received (or local) update
// run — a column-major nrow x ncol block at src (ld), whose row i / column j are rows / columns
// j0 + i / j0 + j of the source's update row set — are added into the owner's panel: entry (i, j),
// i >= j, goes to panels[col[j] + pos[i]] (col = column start inside the destination supernode,
// pos = row position in its rows(P)).  FP64 RED: several sources hit one entry.
struct XTask {
  long long src, col, pos;
  int ld, nrow, c0, nc;
};

constexpr int TILE = 64;           // CTA tile edge (rows and columns)
#ifndef SPCHOL_MINB
#define SPCHOL_MINB 4
#endif
#ifndef SPCHOL_BK
#define SPCHOL_BK 8
#endif
#ifndef SPCHOL_STAGES
#define SPCHOL_STAGES 4
#endif
constexpr int BK = SPCHOL_BK;      // K chunk per pipeline stage
constexpr int STAGES = SPCHOL_STAGES;  // cp.async pipeline depth
constexpr int LDS = TILE + 8;      // smem column stride (doubles): 8 mod 16 -> conflict-free DMMA fragments
constexpr int GEMM_THREADS = 128;  // 4 warps, 2x2, warp tile 32x32
constexpr int GEMM_SMEM = 2 * STAGES * BK * LDS * (int)sizeof(double);
static_assert(GEMM_SMEM >= TILE * (TILE + 4) * (int)sizeof(double), "the epilogue stages the 64x68 tile in the pipeline's shared memory");
constexpr int NBMAX = 64;          // cdiv block width

void launch_gemm(int mode, const GTask* tasks, int ntasks, const SnInfo* sn, double* panels,
                 const double* linv, const long long* ucol_base, const long long* ucol_map,
                 const int* posmap, cudaStream_t st, int prio = 0, int min_smem = 0, int kw_log2 = 0);
void launch_extend_add(const XTask* tasks, int ntasks, const long long* col, const int* pos, double* panels,
                       cudaStream_t st);
#ifndef SPCHOL_TBK
#define SPCHOL_TBK 16
#endif
#ifndef SPCHOL_TSTAGES
#define SPCHOL_TSTAGES 3
#endif
constexpr int TMA_BOX_ROWS = 16;           // 16 doubles = one 128-byte swizzle row
constexpr int TMA_BOX_COLS = SPCHOL_TBK;   // K columns per TMA stage (the host encodes this box)
// TMA variant: tmaps = device array of CUtensorMap (one per supernode panel, rows x columns, box
// 16 x 8, SWIZZLE_128B), tmap_linv = CUtensorMap over the diagonal-inverse slots (64 x 64*slots).
void launch_gemm_tma(int mode, const GTask* tasks, int ntasks, const SnInfo* sn, double* panels, const void* tmaps,
                     const void* tmap_linv, const long long* ucol_base, const long long* ucol_map, const int* posmap,
                     cudaStream_t st, int prio = 0);
void launch_rlb(const RTask* tasks, int ntasks, const SnInfo* sn, double* panels, cudaStream_t st, int prio = 0);
void launch_potrf(const PTask* tasks, int ntasks, const SnInfo* sn, const int* sfirst, double* panels,
                  double* linv, unsigned long long* fail, cudaStream_t st, int prio = 0);
// Fused cdiv of one outer block (columns [c0, c0 + w), w <= 4 * NBMAX) of supernode sn, rows [c0, m)
// cut into 64-row tiles (tile i: rows c0 + 64 i ...; tiles < nbk = ceil(w / 64) hold the diagonal
// blocks).  A task is block (tile, blk), blk < nbk, blk <= tile.  flag = first of the outer block's
// 32 + 4 (ntile - nbk) ready flags (see panel_diag_kernel); slot = inverse slot of inner block 0;
// pw > 0: the task first applies the
// lookahead update by the previous outer block [c0 - pw, c0) (NEXT, K = pw).
struct PanTask {
  int sn, c0, w, tile, blk, slot, flag, pw, q;   // q >= 0: quarter q of the block's NEXT (diagonal region)
};
// One launch = the panel tasks of one outer step over a level's supernodes: the ndiag diagonal-region
// tasks (pair-major: (0,0), (1,0), (1,1), (2,0) ... each pair over all outer blocks), then the
// nbelow blocks below them (column-major: (nbk, 0), (nbk+1, 0), ..., (nbk, 1), ...).  sync3 = {diagonal ticket, below ticket, diagonal CTAs
// done}, zeroed per factor.
// nflags / nslots: sizes of the flag array and of the inverse slots (bounds of the checked build).
void launch_panel(const PanTask* tasks, int ndiag, int nbelow, int* sync3, int* flags, const SnInfo* sn,
                  const int* sfirst, double* panels, double* linv, unsigned long long* fail, int grid_cap,
                  cudaStream_t st, int prio, int nflags, int nslots);
constexpr int SMALL_THREADS = 256;
constexpr int SMALL_MAXK = 64;
constexpr int SMALL_MAXM = SMALL_THREADS;
constexpr int SMALL_MAXELEMS = 12288;   // m*k doubles in shared memory (96 KB)
#ifndef SMALL_DMMA_U
// small_kernel U_J: 2 = DMMA tiles, RED straight from the fragments (default); 1 = DMMA tiles staged
// through shared memory (slower: the staging costs residency); 0 = scalar FMAs
#define SMALL_DMMA_U 2
#endif
// small_kernel shared memory: panel with row stride small_ldp(m) (4 mod 16 doubles: conflict-free
// DMMA fragment loads) and k rounded up to 4 columns, then 8 x 32 doubles of U staging per warp.
__host__ __device__ constexpr int small_ldp(int m) { return (m + 15) / 16 * 16 + 4; }
__host__ __device__ constexpr int small_cta_smem(int m, int k) {
  return small_ldp(m) * ((k + 3) & ~3) + (SMALL_DMMA_U == 1 ? 8 * 256 : 0);
}
constexpr int SMALL_CTA_SMEM_MAX = 16384;   // >= small_cta_smem(m, k) for every m <= 256, m k <= SMALL_MAXELEMS
void launch_small(const int* sns, int count, const SnInfo* sn, const int* sfirst, double* panels,
                  const long long* ucol_base, const long long* ucol_map, const int* posmap, unsigned long long* fail,
                  int smem_doubles, int maxm, int plain, cudaStream_t st, int prio = 0, int maxk = 0);
void launch_init(const double* vals, const long long* amap, long long nnz, double* panels, cudaStream_t st);
// a1 for a subset of A's entries (memory-capped mode: one batch): panels[dst[i]] = vals[idx[i]]
void launch_init_list(const double* vals, const long long* idx, const long long* dst, long long cnt, double* panels,
                      cudaStream_t st);
// Small-supernode solve record (one per supernode, in level / row-class order).
struct SmallSolve {
  long long off, rp;   // panel offset, rows_ptr[J]
  int ld, m, k, f;     // f = first column
};
// rows_class 0 / 1 / 2: m <= 64 / 128 / 256 (rows per lane 2 / 4 / 8)
// Solves run on NR = nr in {1, 2, 4} right-hand sides at once, interleaved: y[i * nr + r].
constexpr int SOLVE_NRMAX = 4;
void launch_solve_small(const SmallSolve* info, int count, int rows_class, int backward, const int* rows,
                        const double* panels, double* y, int nr, cudaStream_t st);
constexpr int SOLVE_THREADS = 256;
constexpr int SOLVE_RCHUNK = 512;   // rows per backward kind-2 task
void launch_solve_fwd_level(const STask* tasks, int ntasks, int* ticket, int* flag, const SnInfo* sn, const int* sfirst,
                            const long long* rows_ptr, const int* rows, const double* panels, const double* linv,
                            double* y, int NB, int nr, cudaStream_t st);
void launch_solve_bwd_level(const STask* tasks, int ntasks, int* ticket, int* flag, int* rcnt, const SnInfo* sn,
                            const int* sfirst, const long long* rows_ptr, const int* rows, const double* panels,
                            const double* linv, double* y, int NB, int nr, cudaStream_t st);
// in: nr columns of n (column-major, ld n) in the caller's order <-> out: interleaved in final order
void launch_permute(const int* perm, const double* in, double* out, long long n, int nr, int inverse, cudaStream_t st);
// multi-GPU solve: as launch_permute, entries whose final row r has mine[r] == 0 become 0
void launch_permute_masked(const int* perm, const unsigned char* mine, const double* in, double* out, long long n,
                           int nr, int inverse, cudaStream_t st);
void launch_axpy(const double* x, double* y, long long n, cudaStream_t st);
void launch_gather(const double* src, const long long* idx, double* out, long long n, cudaStream_t st);
cudaError_t kernels_init_attributes();

}  // namespace spchol
