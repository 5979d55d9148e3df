// sm_100a kernels; see kernels.cuh for the map to the paper.
#include <algorithm>
#include <cstdio>

#include <cuda.h>

#include "kernels.cuh"

namespace spchol {

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// D(8x8) += A(8x4) B(4x8), FP64 tensor core (SASS DMMA.8x8x4).
// Lane (g = lane/4, t = lane%4) holds A[g][t], B[t][g], D[g][2t], D[g][2t+1].
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// Programmatic dependent launch (critical-stream launches, see launch_prio): wait until every
// prerequisite grid has completed and its memory is visible (a no-op for a grid launched without
// the attribute).  The dependents are released implicitly as CTAs exit; releasing them at entry
// (SPCHOL_PDL_EARLY) parks their CTAs on the SMs and measured slower.
__device__ __forceinline__ void pdl_enter() {
#ifdef SPCHOL_PDL_EARLY
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
#endif
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
}

// ----------------------------------------------------------------------------------------------
// gemm_kernel<MODE>: one 64x64 output tile per CTA, C(i,j) = sum_q A(i,q) B(j,q) over q < K, where
// A and B are row blocks of column-major matrices (so both operands stream contiguous columns).
//   MODE_LOCAL   (right-looking update inside supernode J after its block column [c0, c0+nb)):
//                A = panel rows [r0, r0+64), B = panel rows [s0, s0+64), columns [c0, c0+nb), K = nb;
//                panel(row r0+i, col s0+j) -= C(i,j) for r0+i >= s0+j, r0+i < m, s0+j < slot
//                (slot = exclusive column bound of the updated block).
//   MODE_TRSM    A = panel rows [r0, r0+64) x cols [c0, c0+nb), B = L_bb^{-1} (workspace slot), K = nb;
//                panel(r0+i, c0+j) = C(i,j) for r0+i >= s0 (= c0+nb; r0 is rounded down to even)
//                (in place: the CTA owns these rows).
//   MODE_SCATTER A = panel rows [r0, ..), B = panel rows [s0, ..), all k columns (K = k);
//                U(r, c) = C with r = r0+i-k, c = s0+j-k, kept for r >= c >= 0 (lower U_J);
//                ancestor entry address = ucol_base[ucol+c] + posmap[ucol_map[ucol+c] + r0+i]
//                (column start of U's column c inside its ancestor P, then the row's position in
//                rows(P) = m_P-1-relind(J,P)); FP64 RED of -U (concurrent supernodes of
//                one level may hit the same ancestor entry).
// ----------------------------------------------------------------------------------------------
// Shared epilogue of the tile kernels: stage the 64x64 tile through shared memory (column-major,
// stride LDC), then each warp streams whole 64-row columns: 16-byte vector RMW / stores (LOCAL,
// TRSM) or runs of consecutive RED (SCATTER, relind runs are long: consecutive U rows land in
// consecutive ancestor rows).  All destination loads of a thread are issued before its stores.
template <int MODE>
__device__ __forceinline__ void gemm_epilogue(const GTask& T, const SnInfo& S, double* panels, double* smem,
                                              const double (&acc)[4][4][2], const long long* __restrict__ ucol_base,
                                              const long long* __restrict__ ucol_map, const int* __restrict__ posmap) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1, g = lane >> 2, t = lane & 3;
  constexpr int LDC = TILE + 4;   // 68 doubles: conflict-free fragment writes and v2 reads
  double* sC = smem;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int v = 0; v < 2; ++v)
        sC[(wn * 32 + j * 8 + 2 * t + v) * LDC + wm * 32 + i * 8 + g] = acc[i][j][v];
  __syncthreads();
  const int pr = 2 * lane;                 // row pair inside the tile
  constexpr int NIT = TILE / (GEMM_THREADS / 32);   // columns per warp (16)
  if (MODE == MODE_LOCAL) {
    const int gr = T.r0 + pr;
    double2 dv[NIT];
#pragma unroll
    for (int it = 0; it < NIT; ++it) {
      const int gc = T.s0 + warp + 4 * it;
      const bool ok = gc < T.slot && gr + 1 >= gc && gr < S.m;
      dv[it] = ok ? *reinterpret_cast<const double2*>(panels + S.off + (long long)gc * S.ld + gr) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int it = 0; it < NIT; ++it) {
      const int col = warp + 4 * it, gc = T.s0 + col;
      if (!(gc < T.slot && gr + 1 >= gc && gr < S.m)) continue;
      const double2 c2 = *reinterpret_cast<const double2*>(sC + col * LDC + pr);
      double* d = panels + S.off + (long long)gc * S.ld + gr;
      const bool v0 = gr >= gc, v1 = gr + 1 < S.m;
      if (v0 && v1) {
        *reinterpret_cast<double2*>(d) = make_double2(dv[it].x - c2.x, dv[it].y - c2.y);
      } else {
        if (v0) d[0] = dv[it].x - c2.x;
        if (v1) d[1] = dv[it].y - c2.y;
      }
    }
  } else if (MODE == MODE_TRSM) {
    const int gr = T.r0 + pr;
#pragma unroll
    for (int it = 0; it < NIT; ++it) {
      const int col = warp + 4 * it;
      if (col >= T.nb || gr + 1 < T.s0 || gr >= S.m) continue;
      const double2 c2 = *reinterpret_cast<const double2*>(sC + col * LDC + pr);
      double* d = panels + S.off + (long long)(T.c0 + col) * S.ld + gr;
      const bool v0 = gr >= T.s0, v1 = gr + 1 < S.m;
      if (v0 && v1) *reinterpret_cast<double2*>(d) = c2;
      else {
        if (v0) d[0] = c2.x;
        if (v1) d[1] = c2.y;
      }
    }
  } else {
#pragma unroll 4
    for (int it = 0; it < NIT; ++it) {
      const int col = warp + 4 * it;
      const int uc = T.s0 + col - S.k;
      if (uc < 0 || T.s0 + col >= S.m) continue;
      const long long cb = ucol_base[S.ucol + uc];
      const long long mb = ucol_map[S.ucol + uc];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int row = lane + 32 * h, gr = T.r0 + row;   // lanes cover 32 consecutive rows
        if (gr < S.m && gr - S.k >= uc) {
          double* d = panels + cb + posmap[mb + gr];
          if (MODE == MODE_SCATTER_DET) *d -= sC[col * LDC + row];
          else atomicAdd(d, -sC[col * LDC + row]);
        }
      }
    }
  }
}

// RLB epilogue: the block-pair tile is written straight into the ancestor panel at
// dst + j*ldd + i — one relindB per block, no per-row relind lookups; RED because other supernodes
// of the level may update the same ancestor entries.
__device__ __forceinline__ void rlb_epilogue(const RTask& R, double* panels, double* smem, const double (&acc)[4][4][2]) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1, g = lane >> 2, t = lane & 3;
  constexpr int LDC = TILE + 4;
  double* sC = smem;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int v = 0; v < 2; ++v)
        sC[(wn * 32 + j * 8 + 2 * t + v) * LDC + wm * 32 + i * 8 + g] = acc[i][j][v];
  __syncthreads();
  for (int col = R.j0 + warp; col < R.j1; col += GEMM_THREADS / 32) {
    double* d = panels + R.dst + (long long)(col - R.j0) * R.ldd - R.i0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int row = lane + 32 * h;
      if (row >= R.i0 && row < R.i1 && (!R.diag || R.ra + row >= R.rb + col)) atomicAdd(d + row, -sC[col * LDC + row]);
    }
  }
}

template <int MODE>
__global__ void __launch_bounds__(GEMM_THREADS, SPCHOL_MINB) gemm_kernel(const GTask* __restrict__ tasks,
                                                            const SnInfo* __restrict__ sn, double* panels,
                                                            const double* __restrict__ linv,
                                                            const long long* __restrict__ ucol_base,
                                                            const long long* __restrict__ ucol_map,
                                                            const int* __restrict__ posmap, int kw_log2) {
  pdl_enter();
  extern __shared__ __align__(16) double smem[];
  double* sA = smem;
  double* sB = smem + STAGES * BK * LDS;
  GTask T;
  RTask R;
  if (MODE == MODE_RLB) {
    R = reinterpret_cast<const RTask*>(tasks)[blockIdx.x];
    T.sn = R.sn; T.r0 = R.ra; T.s0 = R.rb; T.c0 = 0; T.nb = 0; T.slot = 0;
  } else {
    T = tasks[blockIdx.x];
  }
  const SnInfo S = sn[T.sn];
  const double* A;
  const double* B;
  int lda, ldb, arows, brows, K;
  if (MODE == MODE_LOCAL) {
    A = panels + S.off + (long long)T.c0 * S.ld + T.r0;
    B = panels + S.off + (long long)T.c0 * S.ld + T.s0;
    lda = ldb = S.ld; arows = S.m - T.r0; brows = S.m - T.s0; K = T.nb;
  } else if (MODE == MODE_TRSM) {
    A = panels + S.off + (long long)T.c0 * S.ld + T.r0;
    B = linv + (long long)T.slot * (NBMAX * NBMAX);
    lda = S.ld; ldb = NBMAX; arows = S.m - T.r0; brows = T.nb; K = T.nb;
  } else {   // MODE_SCATTER(_DET / _KS) and MODE_RLB: rows of U_J, all k columns (KS: T.nb owned blocks)
    A = panels + S.off + T.r0;
    B = panels + S.off + T.s0;
    lda = ldb = S.ld; arows = S.m - T.r0; brows = S.m - T.s0;
    K = MODE == MODE_SCATTER_KS ? (T.nb << kw_log2) : S.k;
  }
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1, g = lane >> 2, t = lane & 3;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int nchunks = (K + BK - 1) / BK;
  // Each thread owns NP 16-byte pieces (two rows of one K column) of each operand per chunk; the
  // source pointers and zero-fill sizes are fixed, only the K tail needs a per-chunk check.
  constexpr int NP = (BK * TILE / 2) / GEMM_THREADS;
  const double* srcA[NP];
  const double* srcB[NP];
  int byA[NP], byB[NP], kkp[NP], dofs[NP];
#pragma unroll
  for (int i = 0; i < NP; ++i) {
    const int p = tid + i * GEMM_THREADS;
    const int kk = p >> 5, rp = (p & 31) * 2;
    const int ra = max(0, min(2, arows - rp)), rb = max(0, min(2, brows - rp));
    byA[i] = ra * 8;
    byB[i] = rb * 8;
    srcA[i] = ra ? A + (long long)kk * lda + rp : A;
    srcB[i] = rb ? B + (long long)kk * ldb + rp : B;
    kkp[i] = kk;
    dofs[i] = kk * LDS + rp;
  }
  const long long stepA = (long long)BK * lda, stepB = (long long)BK * ldb;
  auto load_chunk = [&](int chunk, int stage) {
    double* dA = sA + stage * BK * LDS;
    double* dB = sB + stage * BK * LDS;
    if (MODE == MODE_SCATTER_KS) {
      // chunk -> column of the rank's i-th owned block: c0 + i * slot + (chunk mod chunks per block) * BK
      const int cpb_log2 = kw_log2 - (BK == 8 ? 3 : 4);
      const int kcol = T.c0 + (chunk >> cpb_log2) * T.slot + (chunk & ((1 << cpb_log2) - 1)) * BK;
      const long long oa = (long long)kcol * lda;
#pragma unroll
      for (int i = 0; i < NP; ++i) {
        const bool kval = kcol + kkp[i] < S.k;
        cp_async16(dA + dofs[i], kval && byA[i] ? srcA[i] + oa : A, kval ? byA[i] : 0);
        cp_async16(dB + dofs[i], kval && byB[i] ? srcB[i] + oa : B, kval ? byB[i] : 0);
      }
      return;
    }
    const int kc = chunk * BK;
#pragma unroll
    for (int i = 0; i < NP; ++i) {
      const bool kval = kc + kkp[i] < K;
      cp_async16(dA + dofs[i], kval && byA[i] ? srcA[i] + chunk * stepA : A, kval ? byA[i] : 0);
      cp_async16(dB + dofs[i], kval && byB[i] ? srcB[i] + chunk * stepB : B, kval ? byB[i] : 0);
    }
  };
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nchunks) load_chunk(s, s);
    cp_async_commit();
  }
  for (int c = 0; c < nchunks; ++c) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    const int nc = c + STAGES - 1;
    if (nc < nchunks) load_chunk(nc, nc % STAGES);
    cp_async_commit();
    const double* cA = sA + (c % STAGES) * BK * LDS + wm * 32 + g;
    const double* cB = sB + (c % STAGES) * BK * LDS + wn * 32 + g;
#pragma unroll
    for (int ks = 0; ks < BK / 4; ++ks) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        a[i] = cA[(ks * 4 + t) * LDS + i * 8];
        b[i] = cB[(ks * 4 + t) * LDS + i * 8];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j], a[i], b[j]);
    }
  }
  cp_async_wait<0>();
  __syncthreads();
  if (MODE == MODE_RLB) rlb_epilogue(R, panels, smem, acc);
  else gemm_epilogue<MODE>(T, S, panels, smem, acc, ucol_base, ucol_map, posmap);
}

// ----------------------------------------------------------------------------------------------
// gemm_tma_kernel<MODE>: same tile contract and epilogues as gemm_kernel, with the operands moved by
// the Tensor Memory Accelerator: per stage, thread 0 issues 2 x 4 boxes of 16 rows x BK columns
// (cp.async.bulk.tensor, SWIZZLE_128B, out-of-bounds rows/columns zero-filled — ragged tiles and K
// tails need no masking) and the CTA's warps consume them through full/empty mbarriers, no CTA-wide
// barrier in the K loop.  128B swizzle: element (row rw of a 16-row box, column kk) sits at
// kk*128 + (((rw>>1) ^ (kk&7))*16) + (rw&1)*8 bytes.  Lane (g, t) of k-step ks takes K index
// kk = 2ks + (t>>1) + 4(t&1) (any K permutation is valid when A and B share it); with it the 32
// lanes' fragment loads hit 32 distinct banks in 2 wavefronts.
// ----------------------------------------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"((unsigned long long)map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

constexpr int TBK = TMA_BOX_COLS;                       // K columns per stage (multiple of 8 = swizzle atom)
constexpr int TSTAGES = SPCHOL_TSTAGES;
constexpr int TSTAGE_DOUBLES = 2 * TILE * TBK;          // A and B boxes of one stage
constexpr int TMA_SMEM = (TSTAGES * TSTAGE_DOUBLES > TILE * (TILE + 4) ? TSTAGES * TSTAGE_DOUBLES : TILE * (TILE + 4)) *
                             (int)sizeof(double) + 1024;

template <int MODE>
__global__ void __launch_bounds__(GEMM_THREADS, 4) gemm_tma_kernel(const GTask* __restrict__ tasks,
                                                                   const SnInfo* __restrict__ sn, double* panels,
                                                                   const CUtensorMap* __restrict__ tmaps,
                                                                   const CUtensorMap* __restrict__ tmap_linv,
                                                                   const long long* __restrict__ ucol_base,
                                                                   const long long* __restrict__ ucol_map,
                                                                   const int* __restrict__ posmap) {
  pdl_enter();
  extern __shared__ unsigned char tsm_raw[];
  // 1024-byte aligned (128B swizzle atom) stage buffers; offsetting the shared pointer (rather than
  // casting through an integer) keeps the shared address space, so fragment loads stay LDS
  const unsigned sbase = smem_u32(tsm_raw);
  double* smem = reinterpret_cast<double*>(tsm_raw + (((sbase + 1023u) & ~1023u) - sbase));
  __shared__ __align__(8) unsigned long long full[TSTAGES];
  __shared__ int done[TSTAGES];            // warps finished with the stage's current chunk
  const GTask T = tasks[blockIdx.x];
  const SnInfo S = sn[T.sn];
  const CUtensorMap* mapA = tmaps + T.sn;
  const CUtensorMap* mapB = MODE == MODE_TRSM ? tmap_linv : mapA;
  int arow, brow, acol, bcol, K;
  if (MODE == MODE_LOCAL) { arow = T.r0; brow = T.s0; acol = bcol = T.c0; K = T.nb; }
  else if (MODE == MODE_TRSM) { arow = T.r0; brow = 0; acol = T.c0; bcol = T.slot * NBMAX; K = T.nb; }
  else { arow = T.r0; brow = T.s0; acol = bcol = 0; K = S.k; }
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1, g = lane >> 2, t = lane & 3;
  const int nchunks = (K + TBK - 1) / TBK;
  if (tid == 0) {
    for (int s = 0; s < TSTAGES; ++s) { mbar_init(&full[s], 1); done[s] = 0; }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int chunk, int stage) {
    double* dA = smem + stage * TSTAGE_DOUBLES;
    double* dB = dA + TILE * TBK;
    mbar_expect_tx(&full[stage], TSTAGE_DOUBLES * (unsigned)sizeof(double));
#pragma unroll
    for (int q = 0; q < TILE / 16; ++q) {
      tma_load_2d(dA + q * 16 * TBK, mapA, arow + 16 * q, acol + chunk * TBK, &full[stage]);
      tma_load_2d(dB + q * 16 * TBK, mapB, brow + 16 * q, bcol + chunk * TBK, &full[stage]);
    }
  };
  if (tid == 0)
    for (int s = 0; s < TSTAGES && s < nchunks; ++s) issue(s, s);
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  // fragment offsets (doubles) inside a stage, per subtile i and k-step ks (swizzled)
  constexpr int KS = TBK / 4;
  int offA[4][KS], offB[4][KS];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int kk = 8 * (ks >> 1) + 2 * (ks & 1) + (t >> 1) + 4 * (t & 1);
      const int ra = wm * 32 + i * 8 + g, rb = wn * 32 + i * 8 + g;
      offA[i][ks] = (ra >> 4) * 16 * TBK + kk * 16 + ((((ra & 15) >> 1) ^ (kk & 7)) << 1) + (ra & 1);
      offB[i][ks] = TILE * TBK + (rb >> 4) * 16 * TBK + kk * 16 + ((((rb & 15) >> 1) ^ (kk & 7)) << 1) + (rb & 1);
    }
  for (int c = 0; c < nchunks; ++c) {
    const int stage = c % TSTAGES;
    const unsigned parity = (c / TSTAGES) & 1;
    mbar_wait(&full[stage], parity);
    const double* st = smem + stage * TSTAGE_DOUBLES;
    // K tail inside the panel (e.g. a 40-column block): TMA reads real columns there, mask them
    const int kleft = K - c * TBK;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      double a[4], b[4];
      const bool kval = kleft >= TBK || 8 * (ks >> 1) + 2 * (ks & 1) + (t >> 1) + 4 * (t & 1) < kleft;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        a[i] = kval ? st[offA[i][ks]] : 0.0;
        b[i] = kval ? st[offB[i][ks]] : 0.0;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j], a[i], b[j]);
    }
    // the last warp to finish this stage refills it with chunk c + TSTAGES (nobody waits)
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      if (atomicAdd(&done[stage], 1) == GEMM_THREADS / 32 - 1) {
        done[stage] = 0;
        if (c + TSTAGES < nchunks) issue(c + TSTAGES, stage);
      }
    }
  }
  __syncthreads();
  gemm_epilogue<MODE>(T, S, panels, smem, acc, ucol_base, ucol_map, posmap);
}

// ----------------------------------------------------------------------------------------------
// small_kernel: the whole RL step of one small supernode J per CTA (k_J <= 64, m_J <= 256,
// m_J k_J <= SMALL_MAXELEMS), with the panel resident in shared memory:
//   cdiv(J): unblocked right-looking Cholesky of the k x k block + TRSM of the rows below,
//     thread r owns panel row r, two barriers per column;
//   U_J = L_R L_R^T, 4x4 register blocks of the lower t x t update, K = k;
//   assembly: each U entry is RED-added (negated) into its ancestor panel through
//     relind (posmap), exactly as in the tiled scatter kernel.
// Thousands of these supernodes make up the lower levels of the 2D configs.
// ----------------------------------------------------------------------------------------------
__device__ __forceinline__ double rsqrt_nr(double d);

__global__ void __launch_bounds__(SMALL_THREADS) small_kernel(const int* __restrict__ sns,
                                                              const SnInfo* __restrict__ sn,
                                                              const int* __restrict__ sfirst, double* panels,
                                                              const long long* __restrict__ ucol_base,
                                                              const long long* __restrict__ ucol_map,
                                                              const int* __restrict__ posmap,
                                                              unsigned long long* fail, int plain) {
  pdl_enter();
  extern __shared__ double P[];         // k4 x ldp, column-major (ldp = 4 mod 16), columns >= k zero
  const int J = sns[blockIdx.x];
  const SnInfo S = sn[J];
  const int m = S.m, k = S.k, t = m - k, tid = threadIdx.x, ldp = small_ldp(m), k4 = (k + 3) & ~3;
  double* G = panels + S.off;
  // all loads in flight at once (8-byte cp.async; a plain load-store loop serialises the round trips)
  for (int e = tid; e < m * k4; e += blockDim.x) {
    const int c = e / m, r = e - c * m;
    const unsigned sa = (unsigned)__cvta_generic_to_shared(P + c * ldp + r);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa),
                 "l"(c < k ? G + (long long)c * S.ld + r : G), "r"(c < k ? 8 : 0));
  }
  asm volatile("cp.async.wait_all;\n" ::);
  __syncthreads();
  int bad = -1;
  const int r = tid;                      // this thread's panel row
  __shared__ double colbuf[SMALL_MAXM];   // multipliers L(c0.., j) of the current column
  __shared__ double piv;
  // Register-blocked left-looking factor, 8 columns at a time: the row's 8 entries of the block
  // are updated by every earlier column (1 own load + 8 broadcast multipliers per 8 FMAs), then the
  // block is factored right-looking with the pivot and the block rows' multipliers through shared
  // memory (two barriers per column).
  for (int c0 = 0; c0 < k; c0 += 8) {
    double v[8];
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) v[cc] = (r < m && c0 + cc < k4) ? P[(c0 + cc) * ldp + r] : 0.0;
    for (int q = 0; q < c0; ++q) {
      const double l = r < m ? P[q * ldp + r] : 0.0;
#pragma unroll
      for (int cc = 0; cc < 8; ++cc) v[cc] = fma(-l, P[q * ldp + min(c0 + cc, ldp - 1)], v[cc]);
    }
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) {
      const int j = c0 + cc;
      if (j >= k) break;                  // uniform over the CTA
      if (r == j) piv = v[cc];
      __syncthreads();
      const double d = piv;
      const double rl = rsqrt_nr(d);
      if (bad < 0 && !(d > 0.0)) bad = j;
      v[cc] = r > j ? v[cc] * rl : (r == j ? d * rl : 0.0);
      if (r > j && r < c0 + 8) colbuf[r] = v[cc];
      __syncthreads();
#pragma unroll
      for (int c2 = cc + 1; c2 < 8; ++c2) v[c2] = fma(-v[cc], colbuf[min(c0 + c2, SMALL_MAXM - 1)], v[c2]);
    }
#pragma unroll
    for (int cc = 0; cc < 8; ++cc)
      if (r < m && c0 + cc < k) P[(c0 + cc) * ldp + r] = v[cc];
    __syncthreads();
  }
  if (tid == 0 && bad >= 0) atomicMin(fail, (unsigned long long)(sfirst[J] + bad));
  for (int e = tid; e < m * k; e += blockDim.x) {
    const int c = e / m, rr = e - c * m;
    if (rr >= c) G[(long long)c * S.ld + rr] = P[c * ldp + rr];
  }
  if (t <= 0) return;
#if SMALL_DMMA_U
  {
    // U_J = L_R L_R^T on DMMA m8n8k4: work items of 8 U columns x 32 U rows (4 row tiles) dealt to
    // the warps; each is staged per warp in shared memory and RED-scattered column by column with
    // lanes over 32 consecutive U rows (runs of consecutive ancestor rows).  U row r = panel row k + r.
    const int nw = blockDim.x >> 5, warp = tid >> 5, lane = tid & 31, g = lane >> 2, tg = lane & 3;
#if SMALL_DMMA_U == 1
    double* Ust = P + ldp * k4 + warp * 256;
#endif
    const int nt8 = (t + 7) >> 3, nr32 = (t + 31) >> 5;
    int item = 0;
    for (int Jc = 0; Jc < nt8; ++Jc)
      for (int I4 = Jc >> 2; I4 < nr32; ++I4, ++item) {
        if (item % nw != warp) continue;
        double acc[4][2];
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = 0.0;
        const int rb = k + 8 * Jc + g;
        for (int q = 0; q < k4; q += 4) {
          const double b = rb < m ? P[(q + tg) * ldp + rb] : 0.0;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int I = 4 * I4 + i;
            if (8 * I >= t || I < Jc) continue;   // warp-uniform
            const int ra = k + 8 * I + g;
            dmma(acc[i], ra < m ? P[(q + tg) * ldp + ra] : 0.0, b);
          }
        }
#if SMALL_DMMA_U == 2
        {                          // RED straight from the fragments: runs of 8 consecutive U rows
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            const int c = 8 * Jc + 2 * tg + v;
            if (c >= t) continue;
            const long long cbase = ucol_base[S.ucol + c];
            const long long mbase = ucol_map[S.ucol + c];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int ur = 32 * I4 + 8 * i + g;
              if (ur >= t || ur < c) continue;
              double* d = panels + cbase + posmap[mbase + k + ur];
              if (plain) *d -= acc[i][v];
              else atomicAdd(d, -acc[i][v]);
            }
          }
          continue;
        }
#else
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          Ust[(2 * tg) * 32 + 8 * i + g] = acc[i][0];
          Ust[(2 * tg + 1) * 32 + 8 * i + g] = acc[i][1];
        }
        __syncwarp();
        const int ur = 32 * I4 + lane;
#pragma unroll
        for (int c8 = 0; c8 < 8; ++c8) {
          const int c = 8 * Jc + c8;
          if (c >= t) break;
          if (ur < t && ur >= c) {
            const long long cbase = ucol_base[S.ucol + c];
            const long long mbase = ucol_map[S.ucol + c];
            double* d = panels + cbase + posmap[mbase + k + ur];
            if (plain) *d -= Ust[c8 * 32 + lane];
            else atomicAdd(d, -Ust[c8 * 32 + lane]);
          }
        }
        __syncwarp();
#endif
      }
    return;
  }
#else
  // U_J = L_R L_R^T: a work item is (8-column block cb, row r >= 8 cb); consecutive threads take
  // consecutive rows of the same column block, so each RED instruction of a warp covers a run of
  // consecutive U rows of one column = a run of consecutive ancestor rows (coalesced).
  const int ncb = (t + 7) >> 3;
  int item = tid, cb = 0, rows_in_cb = t;
  for (;;) {
    while (cb < ncb && item >= rows_in_cb) { item -= rows_in_cb; ++cb; rows_in_cb = t - 8 * cb; }
    if (cb >= ncb) break;
    const int r = 8 * cb + item;             // U row (panel row k + r)
    const int c0 = 8 * cb;
    double acc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = 0.0;
    for (int p = 0; p < k; ++p) {
      const double lr = P[p * ldp + k + r];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int c = c0 + q;
        const double lc = c < t ? P[p * ldp + k + c] : 0.0;
        acc[q] += lr * lc;
      }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int c = c0 + q;
      if (c >= t || r < c) continue;
      const long long cbase = ucol_base[S.ucol + c];
      const long long mbase = ucol_map[S.ucol + c];
      double* d = panels + cbase + posmap[mbase + k + r];
      if (plain) *d -= acc[q];   // deterministic mode: conflict-free launch
      else atomicAdd(d, -acc[q]);
    }
    item += blockDim.x;
  }
#endif
}

// ----------------------------------------------------------------------------------------------
// small_warp_kernel<R>: the whole RL step of one small supernode per WARP (m_J <= 32 R, k_J <= 64),
// for the bulk of the tiny supernodes of 2D problems (C2: 205K of its 238K supernodes have m <= 64).
// Lane owns panel rows r = lane + 32 i (i < R).  No block barriers: the panel (column-major, ld =
// 32 R) is staged in shared memory by 8-byte cp.async (rows >= m zero-filled), factored
// LEFT-looking column by column (column j = A(:, j) - L(:, 0:j) L(j, 0:j)^T from shared memory,
// the pivot broadcast by shuffle, __syncwarp between columns), written back, then U_J = L_R L_R^T
// is formed on DMMA tiles and RED-scattered through relind (consecutive lanes -> consecutive U
// rows -> mostly consecutive ancestor rows).  A blocked variant (8-column blocks updated by DMMA,
// factored in registers) issued 40% fewer instructions but needed more shared memory per warp and
// measured slower (C2 level 1: 1.81 vs 1.56 ms): the kernel is latency-bound, residency wins.
// ----------------------------------------------------------------------------------------------
__device__ __forceinline__ double rsqrt_nr(double d);

// v[idx][c] with explicit selects (a loop of `if (i == idx)` is turned into an indexed load, which
// puts the whole register array in local memory)
template <int R>
__device__ __forceinline__ double pick_row(const double (&v)[R][8], int idx, int c) {
  if (R == 1) return v[0][c];
  if (R == 2) return idx ? v[R - 1][c] : v[0][c];
  const double lo = (idx & 1) ? v[1][c] : v[0][c];
  const double hi = (idx & 1) ? v[R - 1][c] : v[R > 2 ? 2 : 0][c];
  return (idx & 2) ? hi : lo;
}

template <int R>
__global__ void __launch_bounds__(32) small_warp_kernel(const int* __restrict__ sns, const SnInfo* __restrict__ sn,
                                                        const int* __restrict__ sfirst, double* panels,
                                                        const long long* __restrict__ ucol_base,
                                                        const long long* __restrict__ ucol_map,
                                                        const int* __restrict__ posmap, unsigned long long* fail,
                                                        int plain) {
  pdl_enter();
  constexpr int LD = 32 * R + 4;        // 4 mod 16 doubles: conflict-free DMMA fragment loads
  extern __shared__ double Pw[];        // k4 x LD, column-major (columns >= k zero), then U staging
  const int J = sns[blockIdx.x];
  const SnInfo S = sn[J];
  const int m = S.m, k = S.k, t = m - k, lane = threadIdx.x, k4 = (k + 3) & ~3;
  double* G = panels + S.off;
  for (int c = 0; c < k4; ++c)
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int r = lane + 32 * i;
      const unsigned sa = (unsigned)__cvta_generic_to_shared(Pw + c * LD + r);
      const bool in = r < m && r >= c && c < k;
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(in ? G + (long long)c * S.ld + r : G),
                   "r"(in ? 8 : 0));
    }
  asm volatile("cp.async.wait_all;\n" ::);
  __syncwarp();
  int bad = -1;
  // Register-blocked left-looking factor, 8 columns at a time: the block is updated by every
  // earlier column (per column q: R own-row loads + 8 broadcast multipliers for 8R FMAs), then
  // factored in registers, right-looking, pivots and multipliers broadcast by shuffle.
  for (int c0 = 0; c0 < k; c0 += 8) {
    double v[R][8];
#pragma unroll
    for (int i = 0; i < R; ++i)
#pragma unroll
      for (int cc = 0; cc < 8; ++cc) v[i][cc] = c0 + cc < k ? Pw[(c0 + cc) * LD + lane + 32 * i] : 0.0;
    for (int q = 0; q < c0; ++q) {
      double lr[R], mq[8];
#pragma unroll
      for (int i = 0; i < R; ++i) lr[i] = Pw[q * LD + lane + 32 * i];
#pragma unroll
      for (int cc = 0; cc < 8; ++cc) mq[cc] = Pw[q * LD + min(c0 + cc, LD - 1)];
#pragma unroll
      for (int i = 0; i < R; ++i)
#pragma unroll
        for (int cc = 0; cc < 8; ++cc) v[i][cc] = fma(-lr[i], mq[cc], v[i][cc]);
    }
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) {       // columns >= k (all-zero) only touch columns >= k
      const int j = c0 + cc;
      const double d = __shfl_sync(0xffffffffu, pick_row<R>(v, j >> 5, cc), j & 31);
      const double rl = rsqrt_nr(d);
      if (bad < 0 && j < k && !(d > 0.0)) bad = j;
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const int r = lane + 32 * i;
        v[i][cc] = r > j ? v[i][cc] * rl : (r == j ? d * rl : 0.0);
      }
#pragma unroll
      for (int c2 = cc + 1; c2 < 8; ++c2) {
        const int rc = c0 + c2;            // multiplier L(rc, j): lane rc % 32, slot rc / 32
        const double l = __shfl_sync(0xffffffffu, pick_row<R>(v, rc >> 5, cc), rc & 31);
#pragma unroll
        for (int i = 0; i < R; ++i) v[i][c2] = fma(-v[i][cc], l, v[i][c2]);
      }
    }
#pragma unroll
    for (int i = 0; i < R; ++i)
#pragma unroll
      for (int cc = 0; cc < 8; ++cc)
        if (c0 + cc < k) Pw[(c0 + cc) * LD + lane + 32 * i] = v[i][cc];
    __syncwarp();
  }
  if (lane == 0 && bad >= 0) atomicMin(fail, (unsigned long long)(sfirst[J] + bad));
  for (int c = 0; c < k; ++c)
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int r = lane + 32 * i;
      if (r < m && r >= c) G[(long long)c * S.ld + r] = Pw[c * LD + r];
    }
  if (t <= 0) return;
  // U_J = L_R L_R^T on the FP64 tensor core: per 8-column block Jc, the 8x8 tiles I >= Jc (DMMA
  // m8n8k4 over K = k4), RED-scattered straight from the fragments (runs of 8 consecutive U rows =
  // mostly consecutive ancestor rows; no staging memory, so more warps stay resident).
  // U row r = panel row k + r.
  const int g = lane >> 2, tg = lane & 3, nt8 = (t + 7) >> 3;
  for (int Jc = 0; Jc < nt8; ++Jc) {
    double acc[4 * R][2];
#pragma unroll
    for (int I = 0; I < 4 * R; ++I) acc[I][0] = acc[I][1] = 0.0;
    const int rb = k + 8 * Jc + g;
    for (int q = 0; q < k4; q += 4) {
      const double b = rb < m ? Pw[(q + tg) * LD + rb] : 0.0;
#pragma unroll
      for (int I = 0; I < 4 * R; ++I) {
        if (I < Jc || I >= nt8) continue;   // warp-uniform
        const int ra = k + 8 * I + g;
        dmma(acc[I], ra < m ? Pw[(q + tg) * LD + ra] : 0.0, b);
      }
    }
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      const int c = 8 * Jc + 2 * tg + v;
      if (c >= t) continue;
      const long long cbase = ucol_base[S.ucol + c];
      const long long mbase = ucol_map[S.ucol + c];
#pragma unroll
      for (int I = 0; I < 4 * R; ++I) {
        const int r = 8 * I + g;
        if (I < Jc || I >= nt8 || r >= t || r < c) continue;
        double* d = panels + cbase + posmap[mbase + k + r];
        if (plain) *d -= acc[I][v];       // deterministic mode: conflict-free launch
        else atomicAdd(d, -acc[I][v]);
      }
    }
  }
}

// ----------------------------------------------------------------------------------------------
// 1/sqrt(d) to full FP64 precision: hardware approximation (MUFU.RSQ64H) + two Newton steps;
// shorter dependent chain than rsqrt(double) (which also handles special cases).  d <= 0 or NaN
// gives NaN/inf, which the caller flags as a failed pivot.
__device__ __forceinline__ double rsqrt_nr(double d) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  const double hd = 0.5 * d;
  y = y * fma(-hd * y, y, 1.5);
  y = y * fma(-hd * y, y, 1.5);
  return y;
}

// ----------------------------------------------------------------------------------------------
// potrf9_kernel: cdiv POTRF ("DPOTRF") of one <= 64-column diagonal block in place, plus X =
// L_bb^{-1} into its inverse slot (TRSM-as-GEMM and the solve), the inverse formed alongside the
// factorization.  Right-looking in 8-column
// panels p (b = 8p) on column-major shared copies of A (-> L) and Y = I (-> X):
//   phase 1  TRSM of panel p's rows below the diagonal block (one thread per row, warps 0-1);
//            X_pp = L_pp^{-1} (one thread); Y_i -= L_{i,p-1} X_{p-1} for the rows i >= b (warps 2-3,
//            the right-looking forward substitution of L X = I, "DTRSM" on the identity)
//   phase 2  thread 0: the next diagonal block's update by the panel and its 8x8 factor, in
//            registers (8 pivots); warps 1-3: the rest of the trailing SYRK, and X_p = X_pp Y_p
// so the only sequential part is the 64-pivot chain; the inverse costs no extra phase.  16-byte
// cp.async loads, 16-byte stores.  (Replaces a row-major kernel that formed the inverse by blocked
// doubling after the factor: 22.2 -> 20.8 us per block, one CTA, tools/potrf_probe.cu.)
// ----------------------------------------------------------------------------------------------
constexpr int P9_LD = NBMAX + 2;              // column stride (doubles): even (16-byte rows pairs)
constexpr int POTRF9_THREADS = 128;
constexpr int POTRF9_SMEM = (2 * NBMAX * P9_LD + NBMAX + 64) * (int)sizeof(double);
#ifdef SPCHOL_P9_CLOCKS   // tools/potrf_probe.cu: phase timestamps of thread 0
__device__ long long p9_clocks[64];
#define P9_CLK(i) do { if (threadIdx.x == 0) p9_clocks[i] = clock64(); } while (0)
#define P9_CLKT(t, i) do { if (threadIdx.x == (t)) p9_clocks[i] = clock64(); } while (0)
#else
#define P9_CLK(i) do { } while (0)
#define P9_CLKT(t, i) do { } while (0)
#endif

// 8x8 diagonal block at b: (optionally) its update by the previous panel [bp, bp + 8), then its
// factor, all in one thread's registers; pivots' reciprocals into rl.
template <bool UPD>
__device__ __forceinline__ void p9_diag(double* Ls, double* rl, int b, int nb, int& bad, int bp = 0) {
  double a[8][8];
#pragma unroll
  for (int j = 0; j < 8; ++j)
#pragma unroll
    for (int i = j; i < 8; ++i) a[i][j] = Ls[(b + j) * P9_LD + b + i];
  if (UPD) {   // A_bb -= L_{b,p} L_{b,p}^T (the panel rows just TRSM'd): 36 x 8 independent FMAs
    double l[8][8];
#pragma unroll
    for (int q = 0; q < 8; ++q)
#pragma unroll
      for (int i = 0; i < 8; i += 2) {
        const double2 v = *reinterpret_cast<const double2*>(Ls + (bp + q) * P9_LD + b + i);
        l[i][q] = v.x;
        l[i + 1][q] = v.y;
      }
#pragma unroll
    for (int q = 0; q < 8; ++q)
#pragma unroll
      for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int i = j; i < 8; ++i) a[i][j] = fma(-l[i][q], l[j][q], a[i][j]);
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const double d = a[j][j];
    if (bad < 0 && b + j < nb && !(d > 0.0)) bad = b + j;
    const double r = rsqrt_nr(d);
    a[j][j] = d * r;
    rl[b + j] = r;
#pragma unroll
    for (int i = j + 1; i < 8; ++i) a[i][j] *= r;
#pragma unroll
    for (int q = j + 1; q < 8; ++q)
#pragma unroll
      for (int i = q; i < 8; ++i) a[i][q] = fma(-a[i][j], a[q][j], a[i][q]);
  }
#pragma unroll
  for (int j = 0; j < 8; ++j)
#pragma unroll
    for (int i = j; i < 8; ++i) Ls[(b + j) * P9_LD + b + i] = a[i][j];
}

// 4x4 tile (rows r0.., columns c0..; r0, c0 multiples of 4) of A -= L_p L_p^T, K = panel [b, b+8).
__device__ __forceinline__ void p9_syrk_tile(double* Ls, int b, int r0, int c0) {
  double acc[4][4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const double2 u = *reinterpret_cast<const double2*>(Ls + (c0 + j) * P9_LD + r0);
    const double2 v = *reinterpret_cast<const double2*>(Ls + (c0 + j) * P9_LD + r0 + 2);
    acc[0][j] = u.x; acc[1][j] = u.y; acc[2][j] = v.x; acc[3][j] = v.y;
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const double* col = Ls + (b + q) * P9_LD;
    const double2 r01 = *reinterpret_cast<const double2*>(col + r0), r23 = *reinterpret_cast<const double2*>(col + r0 + 2);
    const double2 c01 = *reinterpret_cast<const double2*>(col + c0), c23 = *reinterpret_cast<const double2*>(col + c0 + 2);
    const double lr[4] = {r01.x, r01.y, r23.x, r23.y}, lc[4] = {c01.x, c01.y, c23.x, c23.y};
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = fma(-lr[i], lc[j], acc[i][j]);
  }
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (r0 + i >= c0 + j) Ls[(c0 + j) * P9_LD + r0 + i] = acc[i][j];   // upper part of diagonal tiles unused
}

// The whole block's factor + inverse by the CTA's 128 threads (POTRF9_SMEM bytes of shared memory at
// p9_smem); potrf9_kernel is the right-looking reference for potrf10 (SPCHOL_POTRF9=1, probe).
__device__ __forceinline__ void potrf9_block(const PTask& T, const SnInfo& S, const int* __restrict__ sfirst,
                                             double* panels, double* linv, unsigned long long* fail, double* p9_smem) {
  double* Ls = p9_smem;                        // A -> L (column-major, lower part used)
  double* Xs = Ls + NBMAX * P9_LD;             // Y = I -> X = L^{-1} (column-major)
  double* rl = Xs + NBMAX * P9_LD;             // 1 / L_jj
  double* Xd = rl + NBMAX;                     // X_pp of the current panel (8 x 8, column-major)
  P9_CLK(0);
  const int nb = T.nb, tid = threadIdx.x, warp = tid >> 5;
  double* P = panels + S.off + (long long)T.c0 * S.ld + T.c0;
  // A's block: 16-byte cp.async of row pairs (rows >= nb zero-filled), Y = I meanwhile
  for (int e = tid; e < NBMAX * NBMAX / 2; e += POTRF9_THREADS) {
    const int c = e >> 5, r = (e & 31) * 2;
    if (c < nb && r < nb) {
      const unsigned sa = (unsigned)__cvta_generic_to_shared(Ls + c * P9_LD + r);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(P + (long long)c * S.ld + r),
                   "r"(r + 1 < nb ? 16 : 8));
    }
    *reinterpret_cast<double2*>(Xs + c * P9_LD + r) = make_double2(r == c ? 1.0 : 0.0, r + 1 == c ? 1.0 : 0.0);
  }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  if (nb < NBMAX)   // padding: identity (pivots 1, no coupling)
    for (int e = tid; e < NBMAX * NBMAX; e += POTRF9_THREADS) {
      const int c = e >> 6, r = e & 63;
      if (c >= nb || r >= nb) Ls[c * P9_LD + r] = r == c ? 1.0 : 0.0;
    }
  __syncthreads();
  P9_CLK(1);
  int bad = -1;
  if (tid == 0) p9_diag<false>(Ls, rl, 0, nb, bad);
  __syncthreads();
  P9_CLK(2);
  for (int p = 0; p < NBMAX / 8; ++p) {
    const int b = 8 * p, t0 = b + 8, nt = NBMAX - t0;
    // ---- phase 1
    if (warp < 2) {
      if (tid < nt) {                          // TRSM: row t0 + tid of panel p
        const int r = t0 + tid;
        double x[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = Ls[(b + j) * P9_LD + r];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
#pragma unroll
          for (int q = 0; q < j; ++q) x[j] = fma(-x[q], Ls[(b + q) * P9_LD + b + j], x[j]);
          x[j] *= rl[b + j];
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) Ls[(b + j) * P9_LD + r] = x[j];
      }
    } else {
      if (tid == POTRF9_THREADS - 1) {         // X_pp = L_pp^{-1}: column-oriented substitution
        double x[8][8];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          x[c][c] = rl[b + c];
#pragma unroll
          for (int r = c + 1; r < 8; ++r) {
            double acc = 0.0;
#pragma unroll
            for (int q = c; q < r; ++q) acc = fma(Ls[(b + q) * P9_LD + b + r], x[q][c], acc);
            x[r][c] = -acc * rl[b + r];
          }
        }
#pragma unroll
        for (int c = 0; c < 8; ++c)
#pragma unroll
          for (int r = 0; r < 8; ++r) Xd[c * 8 + r] = r >= c ? x[r][c] : 0.0;
      }
      if (p > 0) {                             // Y_i -= L_{i,p-1} X_{p-1} (rows i >= b, columns < b)
        const int bp = b - 8, nrc = (NBMAX - b) / 8;   // row chunks of 8
        for (int it = tid - 64; it < b * nrc; it += 64) {
          const int c = it % b, i0 = b + 8 * (it / b);
          double xk[8];
#pragma unroll
          for (int k = 0; k < 8; k += 2) {
            const double2 v = *reinterpret_cast<const double2*>(Xs + c * P9_LD + bp + k);
            xk[k] = v.x; xk[k + 1] = v.y;
          }
          double y[8];
#pragma unroll
          for (int i = 0; i < 8; i += 2) {
            const double2 v = *reinterpret_cast<const double2*>(Xs + c * P9_LD + i0 + i);
            y[i] = v.x; y[i + 1] = v.y;
          }
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const double* lc = Ls + (bp + k) * P9_LD + i0;
#pragma unroll
            for (int i = 0; i < 8; i += 2) {
              const double2 l = *reinterpret_cast<const double2*>(lc + i);
              y[i] = fma(-l.x, xk[k], y[i]);
              y[i + 1] = fma(-l.y, xk[k], y[i + 1]);
            }
          }
#pragma unroll
          for (int i = 0; i < 8; i += 2) *reinterpret_cast<double2*>(Xs + c * P9_LD + i0 + i) = make_double2(y[i], y[i + 1]);
        }
      }
    }
    __syncthreads();
    P9_CLK(3 + 2 * p);
    // ---- phase 2
    if (warp == 0) {
      if (nt > 0) {
        // the next diagonal block: its update by this panel and its factor in thread 0's registers
        P9_CLKT(0, 21 + p);
        if (tid == 0) p9_diag<true>(Ls, rl, t0, nb, bad, b);
        P9_CLKT(0, 29 + p);
      }
    } else {
      if (warp >= 2 && tid - 64 < t0) {        // X_p = X_pp Y_p, column tid - 64 (< b + 8), in place
        const int c = tid - 64;
        double y[8], xo[8];
#pragma unroll
        for (int k = 0; k < 8; k += 2) {
          const double2 v = *reinterpret_cast<const double2*>(Xs + c * P9_LD + b + k);
          y[k] = v.x; y[k + 1] = v.y;
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          double acc = 0.0;
#pragma unroll
          for (int k = 0; k <= r; ++k) acc = fma(Xd[k * 8 + r], y[k], acc);
          xo[r] = acc;
        }
#pragma unroll
        for (int r = 0; r < 8; r += 2) *reinterpret_cast<double2*>(Xs + c * P9_LD + b + r) = make_double2(xo[r], xo[r + 1]);
      }
      P9_CLKT(64, 37 + p);
      if (nt > 0) {
        const int n4 = nt / 4, ntiles = n4 * (n4 + 1) / 2;   // tiles 0-2 = the next diagonal block (warp 0)
        for (int t = tid - 29; t < ntiles; t += POTRF9_THREADS - 32) {
          int ti = (int)((sqrtf(8.0f * t + 1.0f) - 1.0f) * 0.5f);   // t = ti (ti + 1) / 2 + tj
          while (ti * (ti + 1) / 2 > t) --ti;
          while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
          const int tj = t - ti * (ti + 1) / 2;
          p9_syrk_tile(Ls, b, t0 + 4 * ti, t0 + 4 * tj);
        }
      }
      P9_CLKT(32, 45 + p);
      P9_CLKT(64, 53 + p);
    }
    __syncthreads();
    P9_CLK(4 + 2 * p);
  }
  if (tid == 0 && bad >= 0) atomicMin(fail, (unsigned long long)(sfirst[T.sn] + T.c0 + bad));
  // L (lower, r >= c) into the panel; X (lower, zero elsewhere) into the inverse slot
  double* W = linv + (long long)T.slot * (NBMAX * NBMAX);
  for (int e = tid; e < NBMAX * NBMAX / 2; e += POTRF9_THREADS) {
    const int c = e >> 5, r = (e & 31) * 2;
    const double2 l = *reinterpret_cast<const double2*>(Ls + c * P9_LD + r);
    const double2 x = *reinterpret_cast<const double2*>(Xs + c * P9_LD + r);
    const bool in0 = r >= c && r < nb && c < nb, in1 = r + 1 >= c && r + 1 < nb && c < nb;
    *reinterpret_cast<double2*>(W + e * 2) = make_double2(in0 ? x.x : 0.0, in1 ? x.y : 0.0);
    double* d = P + (long long)c * S.ld + r;
    if (in0 && in1) *reinterpret_cast<double2*>(d) = l;
    else {
      if (in0) d[0] = l.x;
      if (in1) d[1] = l.y;
    }
  }
  P9_CLK(20);
}

// ----------------------------------------------------------------------------------------------
// potrf10_block: the same contract as potrf9_block (factor + inverse of one <= 64-column diagonal
// block, "DPOTRF"), restructured so that only the 8x8 pivot factors stay sequential.  Panels p
// of 8 columns (b = 8p), three barrier phases each:
//   1  thread 0: D_p (already updated) -> L_pp, 1/L_jj, X_pp = L_pp^{-1} in registers;
//      warps 1-3 meanwhile, on DMMA: the lookahead update of panel p+1's columns by panels < p
//      (left-looking, K = 8p) and X's row block p-1: X_{p-1,<} = -X_{p-1,p-1} L_{p-1,<} X_{<,<}
//      (L X = I by row blocks)
//   2  TRSM of panel p's rows below: L_{r,p} = A_{r,p} X_pp^T (one thread per row, depth 8)
//   3  panel p+1's columns -= L_{.,p} L_{p+1,p}^T (DMMA, K = 8)
// L in shared memory column-major, X row-major (both stride P10_LD = 72: conflict-free fragments).
// ----------------------------------------------------------------------------------------------
constexpr int P10_LD = 72;
constexpr int POTRF10_SMEM = (2 * NBMAX * P10_LD + NBMAX + 2 * 64 + 8 * 64) * (int)sizeof(double);

__device__ __forceinline__ void bar_sync_n(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
// (potrf10_block synchronises its 128 threads on named barrier 1, so a caller with more threads runs it
// on threads 0-127 only)
template <bool LOAD = true>
__device__ __forceinline__ void potrf10_block(const PTask& T, const SnInfo& S, const int* __restrict__ sfirst,
                                              double* panels, double* linv, unsigned long long* fail, double* smem) {
  double* Ls = smem;                       // L[r][c] at Ls[c * P10_LD + r]
  double* Xs = Ls + NBMAX * P10_LD;        // X[r][c] at Xs[r * P10_LD + c]
  double* rl = Xs + NBMAX * P10_LD;        // 1 / L_jj
  double* Xd = rl + NBMAX;                 // X_pp of panels p (even / odd), row-major 8 x 8 each
  double* Tsc = Xd + 128;                  // 8 x 64 row-major scratch (X row block products)
  const int nb = T.nb, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  constexpr int LD = P10_LD;
  double* P = panels + S.off + (long long)T.c0 * S.ld + T.c0;
  if (LOAD) {
    for (int e = tid; e < NBMAX * NBMAX / 2; e += POTRF9_THREADS) {
      const int c = e >> 5, r = (e & 31) * 2;
      if (c < nb && r < nb && r + 1 >= c) cp_async16(Ls + c * LD + r, P + (long long)c * S.ld + r, r + 1 < nb ? 16 : 8);
    }
    cp_async_commit();
  }
  for (int e = tid; e < NBMAX * LD / 2; e += POTRF9_THREADS) reinterpret_cast<double2*>(Xs)[e] = make_double2(0.0, 0.0);
  if (LOAD) cp_async_wait<0>();
  if (nb < NBMAX) {   // padding: identity (pivots 1, no coupling)
    bar_sync_n(1, POTRF9_THREADS);
    for (int e = tid; e < NBMAX * NBMAX; e += POTRF9_THREADS) {
      const int c = e >> 6, r = e & 63;
      if (c >= nb || r >= nb) Ls[c * LD + r] = r == c ? 1.0 : 0.0;
    }
  }
  bar_sync_n(1, POTRF9_THREADS);
  int bad = -1;
  // X row block pb (rows 8 pb ..): T = L_{pb,<} X_{<,<} on column tile j0, then X = -X_pb,pb T
  auto x_block = [&](int pb, int j0) {
    const int bb = 8 * pb;
    double acc[2] = {0.0, 0.0};
    for (int q = j0; q < bb; q += 4) dmma(acc, Ls[(q + t) * LD + bb + g], Xs[(q + t) * LD + j0 + g]);
    Tsc[g * 64 + j0 + 2 * t] = acc[0];
    Tsc[g * 64 + j0 + 2 * t + 1] = acc[1];
    __syncwarp();
    const double* Xp = Xd + (pb & 1) * 64;
    double x2[2] = {0.0, 0.0};
    dmma(x2, Xp[g * 8 + t], Tsc[t * 64 + j0 + g]);
    dmma(x2, Xp[g * 8 + 4 + t], Tsc[(4 + t) * 64 + j0 + g]);
    Xs[(bb + g) * LD + j0 + 2 * t] = -x2[0];
    Xs[(bb + g) * LD + j0 + 2 * t + 1] = -x2[1];
  };
  // rows r0.. x columns c0..c0+7 of L's trailing part -= L[r0.., q0..q1) L[c0.., q0..q1)^T
  auto upd_tile = [&](int r0, int c0, int q0, int q1) {
    double acc[2] = {Ls[(c0 + 2 * t) * LD + r0 + g], Ls[(c0 + 2 * t + 1) * LD + r0 + g]};
    for (int q = q0; q < q1; q += 4) dmma(acc, -Ls[(q + t) * LD + r0 + g], Ls[(q + t) * LD + c0 + g]);
    Ls[(c0 + 2 * t) * LD + r0 + g] = acc[0];
    Ls[(c0 + 2 * t + 1) * LD + r0 + g] = acc[1];
  };
  for (int p = 0; p < NBMAX / 8; ++p) {
    const int b = 8 * p;
    // ---- phase 1
    if (warp == 0) {
      if (tid == 0) {
        double a[8][8];
#pragma unroll
        for (int j = 0; j < 8; ++j)
#pragma unroll
          for (int i = j; i < 8; ++i) a[i][j] = Ls[(b + j) * LD + b + i];
        double r[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const double d = a[j][j];
          if (bad < 0 && b + j < nb && !(d > 0.0)) bad = b + j;
          r[j] = rsqrt_nr(d);
          a[j][j] = d * r[j];
#pragma unroll
          for (int i = j + 1; i < 8; ++i) a[i][j] *= r[j];
#pragma unroll
          for (int q = j + 1; q < 8; ++q)
#pragma unroll
            for (int i = q; i < 8; ++i) a[i][q] = fma(-a[i][j], a[q][j], a[i][q]);
        }
        double x[8][8];   // X_pp = L_pp^{-1}, column by column (columns independent)
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          x[c][c] = r[c];
#pragma unroll
          for (int i = c + 1; i < 8; ++i) {
            double acc = 0.0;
#pragma unroll
            for (int q = c; q < i; ++q) acc = fma(a[i][q], x[q][c], acc);
            x[i][c] = -acc * r[i];
          }
        }
        double* Xp = Xd + (p & 1) * 64;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          rl[b + j] = r[j];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            if (i >= j) {
              Ls[(b + j) * LD + b + i] = a[i][j];
              Xs[(b + i) * LD + b + j] = x[i][j];
            }
            Xp[i * 8 + j] = i >= j ? x[i][j] : 0.0;
          }
        }
      }
    } else {
      const int nl = 7 - p;                 // lookahead tiles: rows b+8+8u, panel p+1's columns, K = b
      const int nx = p >= 1 ? p - 1 : 0;    // X row block p-1: column tiles 0, 8, .. (p-2)*8
      for (int job = warp - 1; job < nl + nx; job += 3) {
        if (job < nl) upd_tile(b + 8 + 8 * job, b + 8, 0, b);
        else x_block(p - 1, 8 * (job - nl));
      }
    }
    bar_sync_n(1, POTRF9_THREADS);
    if (p == NBMAX / 8 - 1) break;
    // ---- phase 2: TRSM of panel p's rows below its diagonal block
    if (tid < NBMAX - b - 8) {
      const int r = b + 8 + tid;
      const double* Xp = Xd + (p & 1) * 64;
      double a[8], x[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) a[j] = Ls[(b + j) * LD + r];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        double acc = 0.0;
#pragma unroll
        for (int q = 0; q <= j; ++q) acc = fma(a[q], Xp[j * 8 + q], acc);
        x[j] = acc;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) Ls[(b + j) * LD + r] = x[j];
    }
    bar_sync_n(1, POTRF9_THREADS);
    // ---- phase 3: panel p+1's columns by panel p (K = 8)
    for (int u = warp; u < 7 - p; u += 4) upd_tile(b + 8 + 8 * u, b + 8, b, b + 8);
    bar_sync_n(1, POTRF9_THREADS);
  }
  // X row block 7
  for (int job = warp; job < 7; job += 4) x_block(7, 8 * job);
  if (tid == 0 && bad >= 0) atomicMin(fail, (unsigned long long)(sfirst[T.sn] + T.c0 + bad));
  bar_sync_n(1, POTRF9_THREADS);
  // L (lower, r >= c) into the panel; X (lower, zero elsewhere) column-major into the inverse slot
  double* W = linv + (long long)T.slot * (NBMAX * NBMAX);
  for (int e = tid; e < NBMAX * NBMAX / 2; e += POTRF9_THREADS) {
    const int c = e >> 5, r = (e & 31) * 2;
    const double2 l = *reinterpret_cast<const double2*>(Ls + c * LD + r);
    const bool in0 = r >= c && r < nb && c < nb, in1 = r + 1 >= c && r + 1 < nb && c < nb;
    *reinterpret_cast<double2*>(W + e * 2) = make_double2(in0 ? Xs[r * LD + c] : 0.0, in1 ? Xs[(r + 1) * LD + c] : 0.0);
    double* d = P + (long long)c * S.ld + r;
    if (in0 && in1) *reinterpret_cast<double2*>(d) = l;
    else {
      if (in0) d[0] = l.x;
      if (in1) d[1] = l.y;
    }
  }
}

__global__ void __launch_bounds__(POTRF9_THREADS, 2) potrf10_kernel(const PTask* __restrict__ tasks,
                                                                 const SnInfo* __restrict__ sn,
                                                                 const int* __restrict__ sfirst, double* panels,
                                                                 double* linv, unsigned long long* fail) {
  pdl_enter();
  extern __shared__ __align__(16) double p10_smem[];
  const PTask T = tasks[blockIdx.x];
  const SnInfo S = sn[T.sn];
  potrf10_block(T, S, sfirst, panels, linv, fail, p10_smem);
}

__global__ void __launch_bounds__(POTRF9_THREADS, 3) potrf9_kernel(const PTask* __restrict__ tasks,
                                                                const SnInfo* __restrict__ sn,
                                                                const int* __restrict__ sfirst, double* panels,
                                                                double* linv, unsigned long long* fail) {
  pdl_enter();
  extern __shared__ __align__(16) double p9_smem[];
  const PTask T = tasks[blockIdx.x];
  const SnInfo S = sn[T.sn];
  potrf9_block(T, S, sfirst, panels, linv, fail, p9_smem);
}

__global__ void init_scatter_kernel(const double* __restrict__ vals, const long long* __restrict__ amap,
                                    long long nnz, double* panels) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nnz; e += (long long)gridDim.x * blockDim.x) {
    const long long d = amap[e];
    if (d >= 0) panels[d] = vals[e];     // d < 0: entry initialised by another rank (multi-GPU)
  }
}

// Small supernodes (m <= SMALL_MAXM = 256, k <= 64): one warp per supernode, 8 per CTA, described by
// one packed SmallSolve record.  Lane owns rows r = lane + 32 i (i < ROWS, m <= 32 ROWS) in
// registers; x_c travels by shuffle, so the column chain has no barrier and no division
// (reciprocals of the diagonal are formed up front).  Columns go in chunks of CH whose loads are
// issued one chunk ahead (double buffer).
constexpr int SW_WARPS = 8;

template <int ROWS, int CH>
__device__ __forceinline__ void sw_load_cols(double (&Lb)[CH][ROWS], const double* P, int ld, int m, int k, int c0,
                                             int lane) {
#pragma unroll
  for (int j = 0; j < CH; ++j)
#pragma unroll
    for (int i = 0; i < ROWS; ++i) {
      const int r = lane + 32 * i, c = c0 + j;
      Lb[j][i] = (c < k && r > c && r < m) ? P[(long long)c * ld + r] : 0.0;
    }
}

// Right-hand-side blocks: the solve's work vector y holds NR right-hand sides interleaved
// (y[i * NR + r] = component i of right-hand side r), so one pass over L serves all NR of them.
template <int ROWS, int CH, int NR>
__device__ __forceinline__ void sw_fwd_cols(const double (&Lb)[CH][ROWS], double (&v)[ROWS][NR], double dinv0,
                                            double dinv1, int k, int c0, int lane) {
#pragma unroll
  for (int j = 0; j < CH; ++j) {
    const int c = c0 + j;
    if (c >= k) break;
    const bool lo = c < 32;
    const double dc = __shfl_sync(0xffffffffu, lo ? dinv0 : dinv1, c & 31);
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const double xc = __shfl_sync(0xffffffffu, lo ? v[0][r] : v[ROWS > 1 ? 1 : 0][r], c & 31) * dc;
      if (lane == (c & 31)) { if (lo) v[0][r] = xc; else v[ROWS > 1 ? 1 : 0][r] = xc; }
#pragma unroll
      for (int i = 0; i < ROWS; ++i) v[i][r] -= Lb[j][i] * xc;
    }
  }
}

// Forward: y_J := L_JJ^{-1} y_J, then y[rows(J)[r]] -= (L_RJ y_J)_r (RED: ancestors are shared).
template <int ROWS, int NR>
__global__ void __launch_bounds__(32 * SW_WARPS, ROWS >= 4 ? 2 : 3) solve_fwd_small_kernel(const SmallSolve* __restrict__ info, int count,
                                                                        const int* __restrict__ rows,
                                                                        const double* __restrict__ panels, double* y) {
  constexpr int CH = ROWS >= 8 ? 2 : 4;
  const int w = blockIdx.x * SW_WARPS + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (w >= count) return;
  const SmallSolve I = info[w];
  const double* P = panels + I.off;
  double La[CH][ROWS], Lb[CH][ROWS];
  sw_load_cols<ROWS, CH>(La, P, I.ld, I.m, I.k, 0, lane);
  const double dinv0 = lane < I.k ? 1.0 / P[(long long)lane * I.ld + lane] : 0.0;
  const double dinv1 = lane + 32 < I.k ? 1.0 / P[(long long)(lane + 32) * I.ld + lane + 32] : 0.0;
  double v[ROWS][NR];
#pragma unroll
  for (int i = 0; i < ROWS; ++i) {
    const int q = lane + 32 * i;
#pragma unroll
    for (int r = 0; r < NR; ++r) v[i][r] = q < I.k ? y[(long long)(I.f + q) * NR + r] : 0.0;
  }
  for (int c0 = 0; c0 < I.k; c0 += 2 * CH) {
    sw_load_cols<ROWS, CH>(Lb, P, I.ld, I.m, I.k, c0 + CH, lane);
    sw_fwd_cols<ROWS, CH, NR>(La, v, dinv0, dinv1, I.k, c0, lane);
    if (c0 + CH >= I.k) break;
    sw_load_cols<ROWS, CH>(La, P, I.ld, I.m, I.k, c0 + 2 * CH, lane);
    sw_fwd_cols<ROWS, CH, NR>(Lb, v, dinv0, dinv1, I.k, c0 + CH, lane);
  }
  const int* R = rows + I.rp;
#pragma unroll
  for (int i = 0; i < ROWS; ++i) {
    const int q = lane + 32 * i;
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      if (q < I.k) y[(long long)(I.f + q) * NR + r] = v[i][r];
      else if (q < I.m) atomicAdd(y + (long long)R[q] * NR + r, v[i][r]);
    }
  }
}

// Backward: y_J := L_JJ^{-T} (y_J - L_RJ^T y_R).
template <int ROWS, int NR>
__global__ void __launch_bounds__(32 * SW_WARPS, ROWS >= 8 ? 2 : 3) solve_bwd_small_kernel(const SmallSolve* __restrict__ info, int count,
                                                                        const int* __restrict__ rows,
                                                                        const double* __restrict__ panels, double* y) {
  constexpr int CH = ROWS >= 8 ? 2 : 4;
  const int w = blockIdx.x * SW_WARPS + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (w >= count) return;
  const SmallSolve I = info[w];
  const double* P = panels + I.off;
  const int* R = rows + I.rp;
  double yr[ROWS][NR];   // y at the rows below the triangle (final values of the ancestors)
#pragma unroll
  for (int i = 0; i < ROWS; ++i) {
    const int q = lane + 32 * i;
#pragma unroll
    for (int r = 0; r < NR; ++r) yr[i][r] = (q >= I.k && q < I.m) ? y[(long long)R[q] * NR + r] : 0.0;
  }
  // t_c = y_c - sum_{q >= k} L_qc y_q: lane c (and c + 32) keeps t_c
  double t0[NR], t1[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    t0[r] = lane < I.k ? y[(long long)(I.f + lane) * NR + r] : 0.0;
    t1[r] = lane + 32 < I.k ? y[(long long)(I.f + lane + 32) * NR + r] : 0.0;
  }
  const double dinv0 = lane < I.k ? 1.0 / P[(long long)lane * I.ld + lane] : 0.0;
  const double dinv1 = lane + 32 < I.k ? 1.0 / P[(long long)(lane + 32) * I.ld + lane + 32] : 0.0;
  if (I.m > I.k)
    for (int c0 = 0; c0 < I.k; c0 += CH) {
      double sj[CH][NR];
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        const int c = c0 + j;
#pragma unroll
        for (int r = 0; r < NR; ++r) sj[j][r] = 0.0;
#pragma unroll
        for (int i = 0; i < ROWS; ++i) {
          const int q = lane + 32 * i;
          const double l = (c < I.k && q >= I.k && q < I.m) ? P[(long long)c * I.ld + q] : 0.0;
#pragma unroll
          for (int r = 0; r < NR; ++r) sj[j][r] += l * yr[i][r];
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int j = 0; j < CH; ++j)
#pragma unroll
          for (int r = 0; r < NR; ++r) sj[j][r] += __shfl_xor_sync(0xffffffffu, sj[j][r], o);
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        const int c = c0 + j;
        if (c < I.k && lane == (c & 31))
#pragma unroll
          for (int r = 0; r < NR; ++r) { if (c < 32) t0[r] -= sj[j][r]; else t1[r] -= sj[j][r]; }
      }
    }
  // triangle, right-looking transposed: x_c = t_c / L_cc, then t_q -= L_cq x_c for q < c
  for (int c1 = I.k; c1 > 0; c1 -= 8) {   // columns c1-1 .. c1-8
    double L0[8], L1[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int c = c1 - 1 - j;
      L0[j] = (c >= 0 && lane < c) ? P[(long long)lane * I.ld + c] : 0.0;
      L1[j] = (c >= 0 && lane + 32 < c) ? P[(long long)(lane + 32) * I.ld + c] : 0.0;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int c = c1 - 1 - j;
      if (c < 0) break;
      const bool lo = c < 32;
      const double dc = __shfl_sync(0xffffffffu, lo ? dinv0 : dinv1, c & 31);
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        const double xc = __shfl_sync(0xffffffffu, lo ? t0[r] : t1[r], c & 31) * dc;
        if (lane == (c & 31)) { if (lo) t0[r] = xc; else t1[r] = xc; }
        t0[r] -= L0[j] * xc;
        t1[r] -= L1[j] * xc;
      }
    }
  }
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    if (lane < I.k) y[(long long)(I.f + lane) * NR + r] = t0[r];
    if (lane + 32 < I.k) y[(long long)(I.f + lane + 32) * NR + r] = t1[r];
  }
}

// ------------------------------------------------------------------ sync-free level solve (large)
// One launch per level and direction.  CTAs claim tasks in list order through an atomic ticket, so
// every task a CTA waits for was claimed earlier by a running CTA (no deadlock whatever the
// scheduling).  A triangle block publishes x_b in y and then its flag (release); consumers poll
// the flag (acquire) and read x_b through L2 (__ldcg: L1 is not coherent across CTAs).
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void wait_geq(const int* p, int v) {
  while (ld_acquire(p) < v) __nanosleep(32);
}
__device__ __forceinline__ void cp_async8(double* sdst, const double* gsrc) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(a), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

constexpr int XLD = NBMAX + 1;   // padded column stride of the inverse in shared memory (no bank conflicts)

// Stage X = L_bb^{-1} (column-major ld NBMAX in linv) into Xs[c * XLD + r].
__device__ __forceinline__ void stage_inverse(double* Xs, const double* X) {
  for (int e = threadIdx.x; e < NBMAX * NBMAX; e += SOLVE_THREADS) cp_async8(Xs + (e >> 6) * XLD + (e & 63), X + e);
}

// Forward, one level: kind 0 = triangle row block b: x_b = X_b (y_b - sum_{c<b} L_bc x_c);
// kind 1 = rows [q0, q1) below the triangle: y[rows(J)[q]] -= sum_c L_qc x_c.  NR right-hand sides.
// Thread (lane = tid & 63, grp = tid >> 6): row q0 + lane, columns grp + 4j of each block.
template <int NR>
__global__ void __launch_bounds__(SOLVE_THREADS) solve_fwd_level_kernel(
    const STask* __restrict__ tasks, int* ticket, int* flag, const SnInfo* __restrict__ sn,
    const int* __restrict__ sfirst, const long long* __restrict__ rows_ptr, const int* __restrict__ rows,
    const double* __restrict__ panels, const double* __restrict__ linv, double* y, int NB) {
  __shared__ double Xs[NBMAX * XLD];
  __shared__ double xs[NBMAX][NR];
  __shared__ double part[4][NBMAX][NR];
  __shared__ int s_task;
  const int tid = threadIdx.x, lane = tid & 63, grp = tid >> 6;
  if (tid == 0) s_task = atomicAdd(ticket, 1);
  __syncthreads();
  const STask T = tasks[s_task];
  const SnInfo S = sn[T.sn];
  const int f = sfirst[T.sn];
  const int slot0 = T.slot - T.cb;
  const bool tri = T.kind == 0;
  if (tri) stage_inverse(Xs, linv + (long long)T.slot * (NBMAX * NBMAX));
  const int q = T.q0 + lane;
  const bool rowok = q < T.q1;
  const double* Pq = panels + S.off + q;
  const int ncb = tri ? T.cb : T.cbhi;
  double acc[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) acc[r] = 0.0;
  for (int cb = T.cblo; cb < ncb; ++cb) {
    const int nbc = min(NB, S.k - cb * NB);
    const double* Lc = Pq + (long long)(cb * NB) * S.ld;
    double lv[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int c = grp + 4 * j;
      lv[j] = (rowok && c < nbc) ? Lc[(long long)c * S.ld] : 0.0;
    }
    if (tid == 0) wait_geq(flag + slot0 + cb, 1);
    __syncthreads();
    for (int e = tid; e < NBMAX * NR; e += SOLVE_THREADS) {
      const int c = e / NR;
      xs[c][e % NR] = c < nbc ? __ldcg(y + (long long)(f + cb * NB) * NR + e) : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 16; ++j)
#pragma unroll
      for (int r = 0; r < NR; ++r) acc[r] += lv[j] * xs[grp + 4 * j][r];
  }
#pragma unroll
  for (int r = 0; r < NR; ++r) part[grp][lane][r] = acc[r];
  __syncthreads();
  if (tri) {
    const int nb = T.nb, b0 = T.cb * NB;
    for (int e = tid; e < NBMAX * NR; e += SOLVE_THREADS) {
      const int c = e / NR, r = e % NR;
      xs[c][r] = c < nb ? __ldcg(y + (long long)(f + b0) * NR + e) -
                              (part[0][c][r] + part[1][c][r] + part[2][c][r] + part[3][c][r]) : 0.0;
    }
    cp_async_wait_all();
    __syncthreads();
    double s[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) s[r] = 0.0;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int c = grp + 4 * j;
      if (c <= lane && c < nb) {
        const double xv = Xs[c * XLD + lane];
#pragma unroll
        for (int r = 0; r < NR; ++r) s[r] += xv * xs[c][r];
      }
    }
#pragma unroll
    for (int r = 0; r < NR; ++r) part[grp][lane][r] = s[r];
    __syncthreads();
    for (int e = tid; e < nb * NR; e += SOLVE_THREADS) {
      const int c = e / NR, r = e % NR;
      y[(long long)(f + b0) * NR + e] = part[0][c][r] + part[1][c][r] + part[2][c][r] + part[3][c][r];
    }
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      st_release(flag + T.slot, 1);
    }
  } else if (grp == 0 && rowok) {
    const long long yq = (long long)rows[rows_ptr[T.sn] + q] * NR;
#pragma unroll
    for (int r = 0; r < NR; ++r) atomicAdd(y + yq + r, -(part[0][lane][r] + part[1][lane][r] + part[2][lane][r] + part[3][lane][r]));
  }
}

// Backward, one level: kind 2 = y_cb -= L(q0:q1, cb)^T y[rows(J)[q0:q1]] (RED), then count;
// kind 3 = x_cb = X_cb^T (y_cb - sum_{r>cb} L_{r,cb}^T x_r) once all kind-2 chunks of cb are in.
// Thread (lane, grp): row lane of a 64-row chunk, columns grp + 4j; sums reduced over the lanes.
template <int NR>
__global__ void __launch_bounds__(SOLVE_THREADS, NR >= 4 ? 1 : 2) solve_bwd_level_kernel(
    const STask* __restrict__ tasks, int* ticket, int* flag, int* rcnt, const SnInfo* __restrict__ sn,
    const int* __restrict__ sfirst, const long long* __restrict__ rows_ptr, const int* __restrict__ rows,
    const double* __restrict__ panels, const double* __restrict__ linv, double* y, int NB) {
  __shared__ double Xs[NBMAX * XLD];
  __shared__ double xs[NBMAX][NR];
  __shared__ double part[4][NBMAX][NR];
  __shared__ double red[4][16][2][NR];
  __shared__ int s_task;
  const int tid = threadIdx.x, lane = tid & 63, grp = tid >> 6;
  if (tid == 0) s_task = atomicAdd(ticket, 1);
  __syncthreads();
  const STask T = tasks[s_task];
  const SnInfo S = sn[T.sn];
  const int f = sfirst[T.sn];
  const int slot0 = T.slot - T.cb;
  const bool tri = T.kind == 3;
  const int c0 = T.cb * NB, nbc = T.nb;
  const double* P = panels + S.off + (long long)c0 * S.ld;
  if (tri) stage_inverse(Xs, linv + (long long)T.slot * (NBMAX * NBMAX));
  double acc[16][NR];
#pragma unroll
  for (int j = 0; j < 16; ++j)
#pragma unroll
    for (int r = 0; r < NR; ++r) acc[j][r] = 0.0;
  if (!tri) {
    const int* R = rows + rows_ptr[T.sn];
    for (int q = T.q0 + lane; q < T.q1; q += 64) {
      double yv[NR];
      const long long yq = (long long)R[q] * NR;
#pragma unroll
      for (int r = 0; r < NR; ++r) yv[r] = y[yq + r];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int c = grp + 4 * j;
        const double l = c < nbc ? P[(long long)c * S.ld + q] : 0.0;
#pragma unroll
        for (int r = 0; r < NR; ++r) acc[j][r] += l * yv[r];
      }
    }
  } else {
    for (int rb = T.cbhi - 1; rb > T.cb; --rb) {
      const int nbr = min(NB, S.k - rb * NB);
      const int q = rb * NB + lane;
      const bool ok = lane < nbr;
      double lv[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int c = grp + 4 * j;
        lv[j] = (ok && c < nbc) ? P[(long long)c * S.ld + q] : 0.0;
      }
      if (tid == 0) wait_geq(flag + slot0 + rb, 1);
      __syncthreads();
      for (int e = tid; e < NBMAX * NR; e += SOLVE_THREADS) {
        const int c = e / NR;
        xs[c][e % NR] = c < nbr ? __ldcg(y + (long long)(f + rb * NB) * NR + e) : 0.0;
      }
      __syncthreads();
#pragma unroll
      for (int j = 0; j < 16; ++j)
#pragma unroll
        for (int r = 0; r < NR; ++r) acc[j][r] += lv[j] * xs[lane][r];
    }
  }
#pragma unroll
  for (int j = 0; j < 16; ++j)
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      double v = acc[j][r];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if ((tid & 31) == 0) red[grp][j][(tid >> 5) & 1][r] = v;
    }
  __syncthreads();
  if (!tri) {
    for (int e = tid; e < nbc * NR; e += SOLVE_THREADS) {
      const int c = e / NR, r = e % NR;
      atomicAdd(y + (long long)(f + c0) * NR + e, -(red[c & 3][c >> 2][0][r] + red[c & 3][c >> 2][1][r]));
    }
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      atomicAdd(rcnt + T.slot, 1);
    }
    return;
  }
  if (tid == 0 && T.need > 0) wait_geq(rcnt + T.slot, T.need);
  cp_async_wait_all();
  __syncthreads();
  for (int e = tid; e < NBMAX * NR; e += SOLVE_THREADS) {
    const int c = e / NR, r = e % NR;
    xs[c][r] = c < nbc ? __ldcg(y + (long long)(f + c0) * NR + e) - (red[c & 3][c >> 2][0][r] + red[c & 3][c >> 2][1][r]) : 0.0;
  }
  __syncthreads();
  double s[NR];   // x_i = sum_{j >= i} X(j, i) v_j, thread i = lane, j = grp + 4jj
#pragma unroll
  for (int r = 0; r < NR; ++r) s[r] = 0.0;
#pragma unroll
  for (int jj = 0; jj < 16; ++jj) {
    const int j = grp + 4 * jj;
    if (j >= lane && j < nbc) {
      const double xv = Xs[lane * XLD + j];
#pragma unroll
      for (int r = 0; r < NR; ++r) s[r] += xv * xs[j][r];
    }
  }
#pragma unroll
  for (int r = 0; r < NR; ++r) part[grp][lane][r] = s[r];
  __syncthreads();
  for (int e = tid; e < nbc * NR; e += SOLVE_THREADS) {
    const int c = e / NR, r = e % NR;
    y[(long long)(f + c0) * NR + e] = part[0][c][r] + part[1][c][r] + part[2][c][r] + part[3][c][r];
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    st_release(flag + T.slot, 1);
  }
}

// The solve's work vector: NR right-hand sides interleaved in final order, y[pf[i] * NR + r] = b[r * n + i].
__global__ void permute_kernel(const int* __restrict__ perm, const double* __restrict__ in, double* out, long long n,
                               int nr, int inverse) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n * nr; e += (long long)gridDim.x * blockDim.x) {
    const long long i = e % n, r = e / n;
    if (inverse) out[e] = in[(long long)perm[i] * nr + r];   // x[r][i] = z[pf[i]][r]
    else out[(long long)perm[i] * nr + r] = in[e];            // y[pf[i]][r] = b[r][i]
  }
}

__global__ void permute_masked_kernel(const int* __restrict__ perm, const unsigned char* __restrict__ mine,
                                      const double* __restrict__ in, double* out, long long n, int nr, int inverse) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n * nr; e += (long long)gridDim.x * blockDim.x) {
    const long long i = e % n, r = e / n;
    const int q = perm[i];
    if (inverse) out[e] = mine[q] ? in[(long long)q * nr + r] : 0.0;
    else out[(long long)q * nr + r] = mine[q] ? in[e] : 0.0;
  }
}

__global__ void gather_kernel(const double* __restrict__ src, const long long* __restrict__ idx, double* out, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = idx[i] >= 0 ? src[idx[i]] : 0.0;   // idx < 0: entry held by another rank (multi-GPU)
}

// ----------------------------------------------------------------------------------------------
// Fused cdiv of one 256-column outer block [c0, c0 + w) of a large supernode ("DPOTRF" +
// "DTRSM", with the right-looking updates inside the outer block and the lookahead update by the
// previous outer block), as one launch pair instead of ~12 launches.  nbk = ceil(w / 64) inner
// blocks; the rows [c0, m) are cut into 64-row tiles, tile i < nbk holding diagonal block i.
//   panel_diag_kernel  the nbk (nbk + 1) / 2 blocks (i, j <= i) of the diagonal region, one task each:
//     (i, i)  NEXT on the block, A_ii -= L_is L_is^T for s < i - 1, then the critical step fused in
//             shared memory: L_{i,i-1} = A_{i,i-1} X_{i-1}^T, A_ii -= L_{i,i-1} L_{i,i-1}^T, POTRF(i)
//             (factor + inverse X_i) without a round trip through memory
//     (i, j<i) NEXT on the block, A_ij -= L_is L_js^T for s < j, then (j < i - 1) L_ij = A_ij X_j^T
//   panel_below_kernel the blocks (i >= nbk, j < nbk) below it, one task each: NEXT, the updates by
//             the blocks s < j, TRSM.
// Ready flags per outer block, F[4 i + j] (diagonal region): (j < i) 1 = A_ij fully updated, 2 = L_ij
// in memory; (j == i) 1 = L_ii and X_i in memory; F[16 + 4 i + j]: quarters of block (i, j)'s NEXT done
// (the diagonal region's lookahead update runs as four K = 64 tasks per block, RED-accumulated, so
// it costs the chain one short product instead of a K = 256 one); F[32 + 4 (i - nbk) + j] (below):
// 2 = L_ij in memory.  Tasks are claimed through a ticket in an order in which
// every wait is on an earlier task of the same outer block, so neither launch can deadlock whatever
// the residency; the below launch is the programmatic dependent of the diagonal one (released once
// every diagonal CTA is resident) and never waits for tasks it could block.  Operands are read with
// cp.async.cg (L2); results are published with threadfence + st.release.gpu, observed with
// ld.acquire.gpu (as in the level solve).
// ----------------------------------------------------------------------------------------------
#ifdef SPCHOL_PK_CLOCKS   // tools/panel_probe.cu: globaltimer stamps per task
__device__ long long pk_clk[8192][8];
#define PK_T(q, e) do { if (threadIdx.x == 0 && (q) < 8192) { long long t_; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); pk_clk[q][e] = t_; } } while (0)
#else
#define PK_T(q, e) do { } while (0)
#endif

// SPCHOL_PK_CHECK (the bounds-checked test build, `make spchol_check`): every panel task's column
// range, rows, inverse slots and flag indices are checked against the launch's bounds; a violation
// prints the task and traps (the sanitizer substitute on this pool).
#ifdef SPCHOL_PK_CHECK
#define PK_CHECK(cond, T)                                                                                  \
  do {                                                                                                     \
    if (!(cond)) {                                                                                         \
      printf("PK_CHECK failed: %s (sn %d c0 %d w %d tile %d blk %d slot %d flag %d pw %d q %d)\n", #cond, \
             (T).sn, (T).c0, (T).w, (T).tile, (T).blk, (T).slot, (T).flag, (T).pw, (T).q);                \
      __trap();                                                                                            \
    }                                                                                                      \
  } while (0)
#else
#define PK_CHECK(cond, T) do { } while (0)
#endif
__device__ __forceinline__ void pk_check_task(const PanTask& T, const SnInfo& S, int nflags, int nslots) {
  const int nbk = (T.w + NBMAX - 1) / NBMAX, ntile = (S.m - T.c0 + TILE - 1) / TILE;
  PK_CHECK(T.c0 >= 0 && T.w >= 1 && T.w <= 4 * NBMAX && T.c0 + T.w <= S.k && T.c0 % NBMAX == 0, T);
  PK_CHECK(T.tile >= 0 && T.tile < ntile && T.blk >= 0 && T.blk < nbk && (T.tile >= nbk || T.blk <= T.tile), T);
  PK_CHECK(T.slot >= 0 && T.slot + nbk <= nslots, T);
  PK_CHECK(T.flag >= 0 && T.flag + 32 + 4 * max(0, ntile - nbk) <= nflags, T);
  PK_CHECK(T.pw >= 0 && T.c0 - T.pw >= 0 && T.q >= -1 && (T.q < 0 || (T.tile < nbk && NBMAX * T.q < T.pw)), T);
  (void)nbk; (void)ntile; (void)nflags; (void)nslots;
}

// acc = A B^T over K columns: A, B = 64-row blocks of column-major matrices (rows past arows /
// brows and columns past K read as zero); the gemm_kernel pipeline (BK-column chunks, cp.async).
// 128 threads: 4 warps in a 2 x 2 grid of 32 x 32 warp tiles.  256 threads (NT): warps 4-7 form a
// second 2 x 2 grid that takes the odd k-steps of every chunk (two warps per SM sub-partition issue
// DMMA, as a lone CTA on the chain needs), reduced into warps 0-3 through shared memory at the end.
template <int NT = GEMM_THREADS>
__device__ __forceinline__ void pk_reduce(double (&acc)[4][4][2], double* red) {
  if (NT == GEMM_THREADS) return;
  const int tid = threadIdx.x;
  if (tid >= GEMM_THREADS) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int v = 0; v < 2; ++v) red[(i * 8 + j * 2 + v) * GEMM_THREADS + tid - GEMM_THREADS] = acc[i][j][v];
  }
  __syncthreads();
  if (tid < GEMM_THREADS) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int v = 0; v < 2; ++v) acc[i][j][v] += red[(i * 8 + j * 2 + v) * GEMM_THREADS + tid];
  }
  __syncthreads();
}

template <int NT = GEMM_THREADS, int BK = spchol::BK, int STAGES = spchol::STAGES>
__device__ __forceinline__ void pk_mma(const double* A, long long lda, int arows, const double* B, long long ldb,
                                       int brows, int K, double (&acc)[4][4][2], double* smem) {
  double* sA = smem;
  double* sB = smem + STAGES * BK * LDS;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, grp = warp >> 2;
  const int wm = (warp >> 1) & 1, wn = warp & 1, g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int nchunks = (K + BK - 1) / BK;
  constexpr int NP = (BK * TILE / 2) / NT;
  const double* srcA[NP];
  const double* srcB[NP];
  int byA[NP], byB[NP], kkp[NP], dofs[NP];
#pragma unroll
  for (int i = 0; i < NP; ++i) {
    const int p = tid + i * NT;
    const int kk = p >> 5, rp = (p & 31) * 2;
    const int ra = max(0, min(2, arows - rp)), rb = max(0, min(2, brows - rp));
    byA[i] = ra * 8;
    byB[i] = rb * 8;
    srcA[i] = ra ? A + kk * lda + rp : A;
    srcB[i] = rb ? B + kk * ldb + rp : B;
    kkp[i] = kk;
    dofs[i] = kk * LDS + rp;
  }
  auto load_chunk = [&](int chunk, int stage) {
    double* dA = sA + stage * BK * LDS;
    double* dB = sB + stage * BK * LDS;
    const int kc = chunk * BK;
#pragma unroll
    for (int i = 0; i < NP; ++i) {
      const bool kval = kc + kkp[i] < K;
      cp_async16(dA + dofs[i], kval && byA[i] ? srcA[i] + kc * lda : A, kval ? byA[i] : 0);
      cp_async16(dB + dofs[i], kval && byB[i] ? srcB[i] + kc * ldb : B, kval ? byB[i] : 0);
    }
  };
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nchunks) load_chunk(s, s);
    cp_async_commit();
  }
  for (int c = 0; c < nchunks; ++c) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    const int nc = c + STAGES - 1;
    if (nc < nchunks) load_chunk(nc, nc % STAGES);
    cp_async_commit();
    const double* cA = sA + (c % STAGES) * BK * LDS + wm * 32 + g;
    const double* cB = sB + (c % STAGES) * BK * LDS + wn * 32 + g;
#pragma unroll
    for (int ks = 0; ks < BK / 4; ++ks) {
      if (NT > GEMM_THREADS && (ks & 1) != grp) continue;
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        a[i] = cA[(ks * 4 + t) * LDS + i * 8];
        b[i] = cB[(ks * 4 + t) * LDS + i * 8];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j], a[i], b[j]);
    }
  }
  cp_async_wait<0>();
  __syncthreads();
  pk_reduce<NT>(acc, smem);
}

// dst (column-major, leading dimension ld, 16-byte aligned row pairs) := C (sub = false) or -= C
// (sub = true) on rows rlo <= r < nrows, columns c < ncols, and r >= c if lower.  The tile is staged
// through shared memory; each warp streams whole columns (16-byte accesses, loads before stores).
// (NT = 256: the tile is in warps 0-3's accumulators; all eight warps stream it out.)
template <int NT = GEMM_THREADS>
__device__ __forceinline__ void pk_store(const double (&acc)[4][4][2], double* smem, double* dst, long long ld, int rlo,
                                         int nrows, int ncols, bool sub, bool lower, bool red = false) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp >> 1) & 1, wn = warp & 1, g = lane >> 2, t = lane & 3;
  constexpr int LDC = TILE + 4;
  constexpr int NW = NT / 32;
  double* sC = smem;
  if (tid < GEMM_THREADS) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int v = 0; v < 2; ++v) sC[(wn * 32 + j * 8 + 2 * t + v) * LDC + wm * 32 + i * 8 + g] = acc[i][j][v];
  }
  __syncthreads();
  const int pr = 2 * lane;
  constexpr int NIT = TILE / NW;
  double2 dv[NIT];
  if (sub && !red) {
#pragma unroll
    for (int it = 0; it < NIT; ++it) {
      const int col = warp + NW * it;
      const bool ok = col < ncols && pr + 1 >= rlo && pr < nrows && (!lower || pr + 1 >= col);
      dv[it] = ok ? *reinterpret_cast<const double2*>(dst + col * ld + pr) : make_double2(0.0, 0.0);
    }
  }
#pragma unroll
  for (int it = 0; it < NIT; ++it) {
    const int col = warp + NW * it;
    const bool v0 = col < ncols && pr >= rlo && pr < nrows && (!lower || pr >= col);
    const bool v1 = col < ncols && pr + 1 >= rlo && pr + 1 < nrows && (!lower || pr + 1 >= col);
    if (!v0 && !v1) continue;
    double2 c2 = *reinterpret_cast<const double2*>(sC + col * LDC + pr);
    double* d = dst + col * ld + pr;
    if (red) {   // dst -= C by FP64 RED (several tasks accumulate into one block)
      if (v0) atomicAdd(d, -c2.x);
      if (v1) atomicAdd(d + 1, -c2.y);
      continue;
    }
    if (sub) c2 = make_double2(dv[it].x - c2.x, dv[it].y - c2.y);
    if (v0 && v1) *reinterpret_cast<double2*>(d) = c2;
    else if (v0) d[0] = c2.x;
    else d[1] = c2.y;
  }
  __threadfence();
  __syncthreads();
}

__device__ __forceinline__ void pk_wait(const int* f, int v) {
  if (threadIdx.x == 0)
    while (ld_acquire(f) < v) __nanosleep(20);
  __syncthreads();
}
__device__ __forceinline__ void pk_publish(int* f, int v) {
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) st_release(f, v);
}

// Geometry of one panel task: tile i's rows, block j's columns.
struct PkGeo {
  int i, nbk, r0, nrows, nr64;
  double* Pc;   // column c0 of the panel
};
__device__ __forceinline__ PkGeo pk_geo(const PanTask& T, const SnInfo& S, double* panels) {
  PkGeo G;
  G.i = T.tile;
  G.nbk = (T.w + NBMAX - 1) / NBMAX;
  G.r0 = T.c0 + NBMAX * G.i;
  G.nrows = S.m - G.r0;
  G.nr64 = min(G.nrows, TILE);
  G.Pc = panels + S.off + (long long)T.c0 * S.ld;
  return G;
}
// A_{i,j} -= L_{i,q} L_{j,q}^T over the columns [c0 + off, c0 + off + K) (off < 0: the previous outer
// block, NEXT); lower if j == i.
template <int NT = GEMM_THREADS>
__device__ __forceinline__ void pk_update(const PanTask& T, const SnInfo& S, const PkGeo& G, int j, int off, int K,
                                          double* smem, bool red = false) {
  double acc[4][4][2];
  const double* Pq = G.Pc + (long long)off * S.ld;
  const int cj = NBMAX * j;
  PK_CHECK(T.c0 + off >= 0 && K >= 1 && T.c0 + off + K <= S.k && cj < T.w && G.r0 < S.m && T.c0 + cj < S.m, T);
  pk_mma<NT>(Pq + G.r0, S.ld, G.nrows, Pq + T.c0 + cj, S.ld, S.m - (T.c0 + cj), K, acc, smem);
  pk_store<NT>(acc, smem, G.Pc + (long long)cj * S.ld + G.r0, S.ld, 0, G.nr64, min(NBMAX, T.w - cj), true, j == G.i, red);
}
// L_{i,s} = A_{i,s} X_s^T on rows >= rlo of the tile
template <int NT = GEMM_THREADS>
__device__ __forceinline__ void pk_trsm(const PanTask& T, const SnInfo& S, const PkGeo& G, int s, int rlo,
                                        const double* linv, double* smem) {
  double acc[4][4][2];
  const int nbs = min(NBMAX, T.w - NBMAX * s);
  double* Ps = G.Pc + (long long)NBMAX * s * S.ld;
  PK_CHECK(s >= 0 && nbs >= 1 && T.c0 + NBMAX * s + nbs <= S.k && G.r0 < S.m && rlo >= 0, T);
  pk_mma<NT>(Ps + G.r0, S.ld, G.nrows, linv + (long long)(T.slot + s) * (NBMAX * NBMAX), NBMAX, nbs, nbs, acc, smem);
  pk_store<NT>(acc, smem, Ps + G.r0, S.ld, rlo, G.nr64, nbs, false, false);
}

// 64 x 64 column-major block (rows contiguous, leading dimension ld) -> shared memory (stride LDS),
// 16-byte cp.async.
template <int NT = GEMM_THREADS>
__device__ __forceinline__ void pk_stage64(double* dst, const double* src, long long ld) {
  for (int e = threadIdx.x; e < TILE * TILE / 2; e += NT) {
    const int c = e >> 5, r = (e & 31) * 2;
    cp_async16(dst + c * LDS + r, src + c * ld + r, 16);
  }
}
// acc (zeroed here) = sA sB^T over K = 64, both operands in shared memory (stride LDS); with
// skip_upper the warp of the strictly upper quadrant (wm < wn) does nothing.
// (NT = 256: warps 4-7 take k in [32, 64), reduced into warps 0-3 through red, 32 KB of scratch.)
template <int NT = GEMM_THREADS>
__device__ __forceinline__ void pk_mma_smem(const double* sA, const double* sB, double (&acc)[4][4][2], bool skip_upper,
                                            double* red = nullptr) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, grp = warp >> 2;
  const int wm = (warp >> 1) & 1, wn = warp & 1, g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const double* cA = sA + wm * 32 + g;
  const double* cB = sB + wn * 32 + g;
  const int k0 = NT > GEMM_THREADS ? grp * (TILE / 2) : 0, k1 = NT > GEMM_THREADS ? k0 + TILE / 2 : TILE;
#pragma unroll 4
  for (int k = k0; k < k1; k += 4) {
    if (skip_upper && wm < wn) break;
    double a[4], b[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      a[i] = cA[(k + t) * LDS + i * 8];
      b[i] = cB[(k + t) * LDS + i * 8];
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) dmma(acc[i][j], a[i], b[j]);
  }
  pk_reduce<NT>(acc, red);
}

constexpr int PANEL_DIAG_SMEM = POTRF10_SMEM + 2 * TILE * LDS * (int)sizeof(double);
static_assert(2 * TILE * LDS >= 2 * STAGES * BK * LDS && 2 * TILE * LDS >= TILE * (TILE + 4), "pk_mma / pk_store staging");

constexpr int PANEL_DIAG_THREADS = 2 * GEMM_THREADS;   // two 2 x 2 warp grids (K split, see pk_mma)
__global__ void __launch_bounds__(PANEL_DIAG_THREADS, 1) panel_diag_kernel(const PanTask* __restrict__ tasks, int ntasks,
                                                                    int* sync3, int* flags, const SnInfo* __restrict__ sn,
                                                                    const int* __restrict__ sfirst, double* panels,
                                                                    double* linv, unsigned long long* fail, int trigger,
                                                                    int nflags, int nslots) {
  pdl_enter();
  if (trigger) asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  extern __shared__ __align__(16) double smem[];
  double* gsm = smem + POTRF10_SMEM / (int)sizeof(double);   // GEMM staging: sA | sB
  double* sA = gsm;
  double* sB = gsm + TILE * LDS;
  double* Ls = smem;
  __shared__ int s_task;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_task = atomicAdd(sync3, 1);
    __syncthreads();
    const int q = s_task;
    if (q >= ntasks) break;
    PK_T(q, 0);
    const PanTask T = tasks[q];
    const SnInfo S = sn[T.sn];
    pk_check_task(T, S, nflags, nslots);
    PK_CHECK(T.tile < (T.w + NBMAX - 1) / NBMAX, T);
    const PkGeo G = pk_geo(T, S, panels);
    const int i = G.i, j = T.blk;
    int* F = flags + T.flag;
    if (T.q >= 0) {   // ---- a quarter (K = 64) of block (i, j)'s NEXT, RED-accumulated, then counted
      pk_update<PANEL_DIAG_THREADS>(T, S, G, j, -T.pw + NBMAX * T.q, min(NBMAX, T.pw - NBMAX * T.q), gsm, true);
      if (threadIdx.x == 0) atomicAdd(F + 16 + 4 * i + j, 1);
      continue;
    }
    if (T.pw > 0) pk_wait(F + 16 + 4 * i + j, (T.pw + NBMAX - 1) / NBMAX);   // NEXT done by its quarter tasks
    PK_T(q, 1);
    if (j < i) {   // ---- off-diagonal block of the diagonal region
      for (int s = 0; s < j; ++s) {
        pk_wait(F + 4 * i + s, 2);
        pk_wait(F + 4 * j + s, 2);
        pk_update<PANEL_DIAG_THREADS>(T, S, G, j, NBMAX * s, min(NBMAX, T.w - NBMAX * s), gsm);
      }
      if (j == i - 1) {
        pk_publish(F + 4 * i + j, 1);   // the diagonal task i does its TRSM (fused)
      } else {
        pk_wait(F + 5 * j, 1);
        pk_trsm<PANEL_DIAG_THREADS>(T, S, G, j, 0, linv, gsm);
        pk_publish(F + 4 * i + j, 2);
      }
      PK_T(q, 7);
      continue;
    }
    // ---- diagonal block i
    for (int s = 0; s + 1 < i; ++s) {   // A_ii -= L_is L_is^T
      pk_wait(F + 4 * i + s, 2);
      pk_update<PANEL_DIAG_THREADS>(T, S, G, i, NBMAX * s, NBMAX, gsm);
    }
    PK_T(q, 2);
    const int ci = NBMAX * i, nbi = min(NBMAX, T.w - ci);
    const PTask P{T.sn, T.c0 + ci, nbi, T.slot + i};
    if (i >= 1 && nbi == NBMAX && G.nrows >= TILE) {
      const int s = i - 1;
      double* Ps = G.Pc + (long long)NBMAX * s * S.ld;
      pk_wait(F + 4 * i + s, 1);          // A_{i,s} (and A_ii, this task's own) fully updated: prefetch them
      pk_stage64<PANEL_DIAG_THREADS>(sA, Ps + G.r0, S.ld);
      {   // A_ii -> Ls (stride P10_LD), lower row pairs
        const double* Aii = G.Pc + (long long)ci * S.ld + G.r0;
        for (int e = threadIdx.x; e < NBMAX * NBMAX / 2; e += PANEL_DIAG_THREADS) {
          const int c = e >> 5, r = (e & 31) * 2;
          if (r + 1 >= c) cp_async16(Ls + c * P10_LD + r, Aii + c * S.ld + r, 16);
        }
      }
      cp_async_commit();
      pk_wait(F + 5 * s, 1);              // POTRF(s): X_s
      PK_T(q, 3);
      pk_stage64<PANEL_DIAG_THREADS>(sB, linv + (long long)(T.slot + s) * (NBMAX * NBMAX), NBMAX);
      cp_async_commit();
      cp_async_wait<0>();
      __syncthreads();
      double acc[4][4][2];
      double* red = Ls + NBMAX * P10_LD;   // (the POTRF's X area: free until potrf10_block starts)
      pk_mma_smem<PANEL_DIAG_THREADS>(sA, sB, acc, false, red);   // L_{i,s} = A_{i,s} X_s^T (in warps 0-3)
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
      const int wm = (warp >> 1) & 1, wn = warp & 1, g = lane >> 2, t = lane & 3;
      if (warp < 4) {
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b)
#pragma unroll
            for (int v = 0; v < 2; ++v) sA[(wn * 32 + b * 8 + 2 * t + v) * LDS + wm * 32 + a * 8 + g] = acc[a][b][v];
      }
      __syncthreads();
      for (int c = warp; c < NBMAX; c += PANEL_DIAG_THREADS / 32)   // L_{i,s} -> panel (published below)
        *reinterpret_cast<double2*>(Ps + (long long)c * S.ld + G.r0 + 2 * lane) =
            *reinterpret_cast<const double2*>(sA + c * LDS + 2 * lane);
      PK_T(q, 4);
      // A_ii -= L_{i,s} L_{i,s}^T (lower quadrants) while the stores drain; L_{i,s}'s consumers (the
      // blocks below, off the critical path) see it after the SYRK
      pk_mma_smem<PANEL_DIAG_THREADS>(sA, sA, acc, true, red);
      if (warp < 4 && wm >= wn) {
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
              const int r = wm * 32 + a * 8 + g, c = wn * 32 + b * 8 + 2 * t + v;
              if (r >= c) Ls[c * P10_LD + r] -= acc[a][b][v];
            }
      }
      pk_publish(F + 4 * i + s, 2);
      PK_T(q, 5);
      if (threadIdx.x < POTRF9_THREADS) potrf10_block<false>(P, S, sfirst, panels, linv, fail, smem);
    } else {
      if (i >= 1) {   // the critical step through memory (partial block or short tile)
        const int s = i - 1;
        pk_wait(F + 4 * i + s, 1);
        pk_wait(F + 5 * s, 1);
        pk_trsm<PANEL_DIAG_THREADS>(T, S, G, s, 0, linv, gsm);
        pk_publish(F + 4 * i + s, 2);
        pk_update<PANEL_DIAG_THREADS>(T, S, G, i, NBMAX * s, NBMAX, gsm);
      }
      if (threadIdx.x < POTRF9_THREADS) potrf10_block<true>(P, S, sfirst, panels, linv, fail, smem);
      if (nbi < NBMAX && G.nrows > nbi) {   // block narrower than the tile: TRSM of the rows below it
        __threadfence();
        __syncthreads();
        pk_trsm<PANEL_DIAG_THREADS>(T, S, G, i, nbi, linv, gsm);
      }
    }
    pk_publish(F + 5 * i, 1);
    PK_T(q, 6);
  }
  // this CTA's work is in memory: count it (panel_below_kernel does not finish before all of them)
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(sync3 + 2, 1);
  }
}

// Blocks (i, j) below the diagonal region (tile i >= nbk, j < nbk), one task each: NEXT on the
// block (independent of the chain), A_ij -= L_is L_js^T for s < j (after (i, s) and the diagonal
// region's (j, s) are published), then L_ij = A_ij X_j^T after POTRF(j); flag F[32 + 4 (i - nbk) + j].
// Launched as the programmatic dependent of panel_diag_kernel WITHOUT griddepcontrol.wait (it
// synchronises through the flags, and only waits for diagonal-kernel tasks or its own earlier
// tasks); it finishes only after every diagonal CTA has counted itself out, so the launch after it
// (whose griddepcontrol.wait covers only this grid) sees all of the outer block's results.
__global__ void __launch_bounds__(GEMM_THREADS, 4) panel_below_kernel(const PanTask* __restrict__ tasks, int ntasks,
                                                                     int* sync3, int ndiag_ctas, int* flags,
                                                                     const SnInfo* __restrict__ sn, double* panels,
                                                                     const double* __restrict__ linv, int nflags, int nslots) {
  extern __shared__ __align__(16) double smem[];
  __shared__ int s_task;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_task = atomicAdd(sync3 + 1, 1);
    __syncthreads();
    const int q = s_task;
    if (q >= ntasks) break;
    PK_T(4096 + q, 0);
    const PanTask T = tasks[q];
    const SnInfo S = sn[T.sn];
    pk_check_task(T, S, nflags, nslots);
    PK_CHECK(T.tile >= (T.w + NBMAX - 1) / NBMAX && T.q < 0, T);
    const PkGeo G = pk_geo(T, S, panels);
    const int j = T.blk;
    int* F = flags + T.flag;
    int* Fi = F + 32 + 4 * (G.i - G.nbk);
    if (T.pw > 0) pk_update(T, S, G, j, -T.pw, T.pw, smem);
    PK_T(4096 + q, 1);
    for (int s = 0; s < j; ++s) {
      pk_wait(Fi + s, 2);
      pk_wait(F + 4 * j + s, 2);
      pk_update(T, S, G, j, NBMAX * s, NBMAX, smem);
    }
    pk_wait(F + 5 * j, 1);
    pk_trsm(T, S, G, j, 0, linv, smem);
    if (j + 1 < G.nbk) pk_publish(Fi + j, 2);
    PK_T(4096 + q, 2);
  }
  if (threadIdx.x == 0)
    while (ld_acquire(sync3 + 2) < ndiag_ctas) __nanosleep(64);
}

// ---------------------------------------------------------------------------------------------- launchers
cudaError_t kernels_init_attributes() {
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(potrf9_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, POTRF9_SMEM))) return e;
  if ((e = cudaFuncSetAttribute(potrf10_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, POTRF10_SMEM))) return e;
  if ((e = cudaFuncSetAttribute(panel_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, PANEL_DIAG_SMEM))) return e;
  if ((e = cudaFuncSetAttribute(panel_below_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, GEMM_SMEM))) return e;
  if ((e = cudaFuncSetAttribute(small_warp_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, ((32 * 1 + 4) * SMALL_MAXK + 8 * 32 * 1) * 8))) return e;
  if ((e = cudaFuncSetAttribute(small_warp_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, ((32 * 2 + 4) * SMALL_MAXK + 8 * 32 * 2) * 8))) return e;
  if ((e = cudaFuncSetAttribute(small_warp_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, ((32 * 4 + 4) * SMALL_MAXK + 8 * 32 * 4) * 8))) return e;
  if ((e = cudaFuncSetAttribute(small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMALL_CTA_SMEM_MAX * (int)sizeof(double)))) return e;
  if ((e = cudaFuncSetAttribute(gemm_kernel<MODE_LOCAL>, cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024))) return e;
  if ((e = cudaFuncSetAttribute(gemm_kernel<MODE_RLB>, cudaFuncAttributeMaxDynamicSharedMemorySize, GEMM_SMEM))) return e;
  if ((e = cudaFuncSetAttribute(gemm_tma_kernel<MODE_LOCAL>, cudaFuncAttributeMaxDynamicSharedMemorySize, TMA_SMEM))) return e;
  if ((e = cudaFuncSetAttribute(gemm_tma_kernel<MODE_TRSM>, cudaFuncAttributeMaxDynamicSharedMemorySize, TMA_SMEM))) return e;
  if ((e = cudaFuncSetAttribute(gemm_tma_kernel<MODE_SCATTER>, cudaFuncAttributeMaxDynamicSharedMemorySize, TMA_SMEM))) return e;
  if ((e = cudaFuncSetAttribute(gemm_kernel<MODE_TRSM>, cudaFuncAttributeMaxDynamicSharedMemorySize, GEMM_SMEM))) return e;
  if ((e = cudaFuncSetAttribute(gemm_kernel<MODE_SCATTER>, cudaFuncAttributeMaxDynamicSharedMemorySize, GEMM_SMEM))) return e;
  if ((e = cudaFuncSetAttribute(gemm_kernel<MODE_SCATTER_DET>, cudaFuncAttributeMaxDynamicSharedMemorySize, GEMM_SMEM))) return e;
  if ((e = cudaFuncSetAttribute(gemm_kernel<MODE_SCATTER_KS>, cudaFuncAttributeMaxDynamicSharedMemorySize, GEMM_SMEM))) return e;
  return cudaSuccess;
}

// Launch with an explicit scheduling priority (cudaLaunchAttributePriority is recorded into the
// kernel node under graph capture; stream priorities alone are not).
static bool pdl_enabled() { const char* e = getenv("SPCHOL_PDL"); return !e || atoi(e) != 0; }   // read per launch
template <typename... KArgs, typename... Args>
static void launch_prio(void (*kern)(KArgs...), int grid, int block, int smem, cudaStream_t st, int prio,
                        Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributePriority;
  attr[0].val.priority = prio;
  // critical-stream launches (high priority): programmatic dependent launch, so the next kernel of
  // the cdiv chain is scheduled while this one runs and only waits for its completion (pdl_enter)
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (prio < 0 && pdl_enabled()) ? 2 : 1;
  cudaLaunchKernelEx(&cfg, kern, args...);
}

void launch_gemm_tma(int mode, const GTask* tasks, int ntasks, const SnInfo* sn, double* panels, const void* tmaps,
                     const void* tmap_linv, const long long* ucol_base, const long long* ucol_map, const int* posmap,
                     cudaStream_t st, int prio) {
  if (ntasks <= 0) return;
  const CUtensorMap* tm = (const CUtensorMap*)tmaps;
  const CUtensorMap* tl = (const CUtensorMap*)tmap_linv;
  if (mode == MODE_LOCAL)
    launch_prio(gemm_tma_kernel<MODE_LOCAL>, ntasks, GEMM_THREADS, TMA_SMEM, st, prio, tasks, sn, panels, tm, tl, ucol_base, ucol_map, posmap);
  else if (mode == MODE_TRSM)
    launch_prio(gemm_tma_kernel<MODE_TRSM>, ntasks, GEMM_THREADS, TMA_SMEM, st, prio, tasks, sn, panels, tm, tl, ucol_base, ucol_map, posmap);
  else
    launch_prio(gemm_tma_kernel<MODE_SCATTER>, ntasks, GEMM_THREADS, TMA_SMEM, st, prio, tasks, sn, panels, tm, tl, ucol_base, ucol_map, posmap);
}

void launch_gemm(int mode, const GTask* tasks, int ntasks, const SnInfo* sn, double* panels, const double* linv,
                 const long long* ucol_base, const long long* ucol_map, const int* posmap, cudaStream_t st, int prio,
                 int min_smem, int kw_log2) {
  if (ntasks <= 0) return;
  if (mode == MODE_LOCAL)
    launch_prio(gemm_kernel<MODE_LOCAL>, ntasks, GEMM_THREADS, std::max(GEMM_SMEM, min_smem), st, prio, tasks, sn, panels, linv, ucol_base, ucol_map, posmap, 0);
  else if (mode == MODE_TRSM)
    launch_prio(gemm_kernel<MODE_TRSM>, ntasks, GEMM_THREADS, GEMM_SMEM, st, prio, tasks, sn, panels, linv, ucol_base, ucol_map, posmap, 0);
  else if (mode == MODE_SCATTER_DET)
    launch_prio(gemm_kernel<MODE_SCATTER_DET>, ntasks, GEMM_THREADS, GEMM_SMEM, st, prio, tasks, sn, panels, linv, ucol_base, ucol_map, posmap, 0);
  else if (mode == MODE_SCATTER_KS)
    launch_prio(gemm_kernel<MODE_SCATTER_KS>, ntasks, GEMM_THREADS, GEMM_SMEM, st, prio, tasks, sn, panels, linv, ucol_base, ucol_map, posmap, kw_log2);
  else
    launch_prio(gemm_kernel<MODE_SCATTER>, ntasks, GEMM_THREADS, GEMM_SMEM, st, prio, tasks, sn, panels, linv, ucol_base, ucol_map, posmap, 0);
}

// Extend-add of the multi-GPU exchange (see XTask): one CTA per task, a warp per column, lanes over
// consecutive rows (coalesced reads of the run, runs of consecutive destination rows).
__global__ void __launch_bounds__(256) extend_add_kernel(const XTask* __restrict__ tasks, const long long* __restrict__ col,
                                                         const int* __restrict__ pos, double* panels) {
  const XTask T = tasks[blockIdx.x];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c = warp; c < T.nc; c += 8) {
    const int j = T.c0 + c;
    const double* s = panels + T.src + (long long)j * T.ld;
    double* d = panels + col[T.col + j];
    const int* p = pos + T.pos;
    for (int i = j + lane; i < T.nrow; i += 32) {
      const double v = s[i];
      if (v != 0.0) atomicAdd(d + p[i], v);
    }
  }
}
void launch_extend_add(const XTask* tasks, int ntasks, const long long* col, const int* pos, double* panels,
                       cudaStream_t st) {
  if (ntasks > 0) extend_add_kernel<<<ntasks, 256, 0, st>>>(tasks, col, pos, panels);
}

void launch_rlb(const RTask* tasks, int ntasks, const SnInfo* sn, double* panels, cudaStream_t st, int prio) {
  if (ntasks <= 0) return;
  launch_prio(gemm_kernel<MODE_RLB>, ntasks, GEMM_THREADS, GEMM_SMEM, st, prio, reinterpret_cast<const GTask*>(tasks), sn,
              panels, (const double*)nullptr, (const long long*)nullptr, (const long long*)nullptr, (const int*)nullptr, 0);
}

void launch_potrf(const PTask* tasks, int ntasks, const SnInfo* sn, const int* sfirst, double* panels, double* linv,
                  unsigned long long* fail, cudaStream_t st, int prio) {
  if (ntasks <= 0) return;
  const bool p9 = getenv("SPCHOL_POTRF9") && atoi(getenv("SPCHOL_POTRF9")) != 0;   // read per launch (tests)
  if (p9) launch_prio(potrf9_kernel, ntasks, POTRF9_THREADS, POTRF9_SMEM, st, prio, tasks, sn, sfirst, panels, linv, fail);
  else launch_prio(potrf10_kernel, ntasks, POTRF9_THREADS, POTRF10_SMEM, st, prio, tasks, sn, sfirst, panels, linv, fail);
}

void launch_panel(const PanTask* tasks, int ndiag, int nbelow, int* sync3, int* flags, const SnInfo* sn,
                  const int* sfirst, double* panels, double* linv, unsigned long long* fail, int grid_cap,
                  cudaStream_t st, int prio, int nflags, int nslots) {
  if (ndiag <= 0) return;
  const int gd = std::min(ndiag, 148);
  launch_prio(panel_diag_kernel, gd, PANEL_DIAG_THREADS, PANEL_DIAG_SMEM, st, prio, tasks, ndiag, sync3, flags, sn, sfirst,
              panels, linv, fail, nbelow > 0 ? 1 : 0, nflags, nslots);
  if (nbelow <= 0) return;
  const int gb = std::min(nbelow, grid_cap > 0 ? grid_cap : 4 * 148);
  launch_prio(panel_below_kernel, gb, GEMM_THREADS, GEMM_SMEM, st, prio, tasks + ndiag, nbelow, sync3, gd, flags, sn,
              panels, (const double*)linv, nflags, nslots);
}

void launch_small(const int* sns, int count, const SnInfo* sn, const int* sfirst, double* panels,
                  const long long* ucol_base, const long long* ucol_map, const int* posmap, unsigned long long* fail,
                  int smem_doubles, int maxm, int plain, cudaStream_t st, int prio, int maxk) {
  if (count <= 0) return;
  if (maxk > 0 && maxm <= 128) {   // one warp per supernode
    const int R = maxm <= 32 ? 1 : (maxm <= 64 ? 2 : 4);
    const int sm = (32 * R + 4) * ((maxk + 3) & ~3) * (int)sizeof(double);
    if (R == 1) launch_prio(small_warp_kernel<1>, count, 32, sm, st, prio, sns, sn, sfirst, panels, ucol_base, ucol_map, posmap, fail, plain);
    else if (R == 2) launch_prio(small_warp_kernel<2>, count, 32, sm, st, prio, sns, sn, sfirst, panels, ucol_base, ucol_map, posmap, fail, plain);
    else launch_prio(small_warp_kernel<4>, count, 32, sm, st, prio, sns, sn, sfirst, panels, ucol_base, ucol_map, posmap, fail, plain);
    return;
  }
  // one thread per panel row: blockDim = the launch's largest m rounded up to a warp (<= 256)
  const int threads = std::min(SMALL_THREADS, std::max(32, (maxm + 31) / 32 * 32));
  launch_prio(small_kernel, count, threads, smem_doubles * (int)sizeof(double), st, prio, sns, sn, sfirst, panels,
              ucol_base, ucol_map, posmap, fail, plain);
}

__global__ void init_list_kernel(const double* __restrict__ vals, const long long* __restrict__ idx,
                                 const long long* __restrict__ dst, long long cnt, double* panels) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < cnt; e += (long long)gridDim.x * blockDim.x)
    panels[dst[e]] = vals[idx[e]];
}
void launch_init_list(const double* vals, const long long* idx, const long long* dst, long long cnt, double* panels,
                      cudaStream_t st) {
  if (cnt <= 0) return;
  long long blocks = (cnt + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  init_list_kernel<<<(int)blocks, 256, 0, st>>>(vals, idx, dst, cnt, panels);
}
void launch_init(const double* vals, const long long* amap, long long nnz, double* panels, cudaStream_t st) {
  if (nnz <= 0) return;
  long long blocks = (nnz + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  init_scatter_kernel<<<(int)blocks, 256, 0, st>>>(vals, amap, nnz, panels);
}

void launch_solve_fwd_level(const STask* tasks, int ntasks, int* ticket, int* flag, const SnInfo* sn, const int* sfirst,
                            const long long* rows_ptr, const int* rows, const double* panels, const double* linv,
                            double* y, int NB, int nr, cudaStream_t st) {
  if (ntasks <= 0) return;
  auto k = nr == 4 ? solve_fwd_level_kernel<4> : nr == 2 ? solve_fwd_level_kernel<2> : solve_fwd_level_kernel<1>;
  k<<<ntasks, SOLVE_THREADS, 0, st>>>(tasks, ticket, flag, sn, sfirst, rows_ptr, rows, panels, linv, y, NB);
}
void launch_solve_bwd_level(const STask* tasks, int ntasks, int* ticket, int* flag, int* rcnt, const SnInfo* sn,
                            const int* sfirst, const long long* rows_ptr, const int* rows, const double* panels,
                            const double* linv, double* y, int NB, int nr, cudaStream_t st) {
  if (ntasks <= 0) return;
  auto k = nr == 4 ? solve_bwd_level_kernel<4> : nr == 2 ? solve_bwd_level_kernel<2> : solve_bwd_level_kernel<1>;
  k<<<ntasks, SOLVE_THREADS, 0, st>>>(tasks, ticket, flag, rcnt, sn, sfirst, rows_ptr, rows, panels, linv, y, NB);
}
template <int NR>
static void solve_small_nr(const SmallSolve* info, int count, int rows_class, int backward, const int* rows,
                           const double* panels, double* y, cudaStream_t st) {
  const int grid = (count + SW_WARPS - 1) / SW_WARPS, thr = 32 * SW_WARPS;
  if (!backward) {
    if (rows_class == 0) solve_fwd_small_kernel<2, NR><<<grid, thr, 0, st>>>(info, count, rows, panels, y);
    else if (rows_class == 1) solve_fwd_small_kernel<4, NR><<<grid, thr, 0, st>>>(info, count, rows, panels, y);
    else solve_fwd_small_kernel<8, NR><<<grid, thr, 0, st>>>(info, count, rows, panels, y);
  } else {
    if (rows_class == 0) solve_bwd_small_kernel<2, NR><<<grid, thr, 0, st>>>(info, count, rows, panels, y);
    else if (rows_class == 1) solve_bwd_small_kernel<4, NR><<<grid, thr, 0, st>>>(info, count, rows, panels, y);
    else solve_bwd_small_kernel<8, NR><<<grid, thr, 0, st>>>(info, count, rows, panels, y);
  }
}
void launch_solve_small(const SmallSolve* info, int count, int rows_class, int backward, const int* rows,
                        const double* panels, double* y, int nr, cudaStream_t st) {
  if (count <= 0) return;
  if (nr == 4) solve_small_nr<4>(info, count, rows_class, backward, rows, panels, y, st);
  else if (nr == 2) solve_small_nr<2>(info, count, rows_class, backward, rows, panels, y, st);
  else solve_small_nr<1>(info, count, rows_class, backward, rows, panels, y, st);
}
__global__ void axpy_kernel(const double* __restrict__ x, double* y, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    y[i] += x[i];
}
void launch_axpy(const double* x, double* y, long long n, cudaStream_t st) {
  if (n <= 0) return;
  long long blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  axpy_kernel<<<(int)blocks, 256, 0, st>>>(x, y, n);
}
void launch_gather(const double* src, const long long* idx, double* out, long long n, cudaStream_t st) {
  if (n <= 0) return;
  long long blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  gather_kernel<<<(int)blocks, 256, 0, st>>>(src, idx, out, n);
}
void launch_permute(const int* perm, const double* in, double* out, long long n, int nr, int inverse, cudaStream_t st) {
  if (n <= 0) return;
  long long blocks = (n * nr + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  permute_kernel<<<(int)blocks, 256, 0, st>>>(perm, in, out, n, nr, inverse);
}
void launch_permute_masked(const int* perm, const unsigned char* mine, const double* in, double* out, long long n,
                           int nr, int inverse, cudaStream_t st) {
  if (n <= 0) return;
  long long blocks = (n * nr + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  permute_masked_kernel<<<(int)blocks, 256, 0, st>>>(perm, mine, in, out, n, nr, inverse);
}

}  // namespace spchol
