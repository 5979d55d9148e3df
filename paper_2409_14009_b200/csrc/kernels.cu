// sm_100a kernels; see kernels.cuh for the map to the paper.
#include <cstdio>

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
template <int MODE>
__global__ void __launch_bounds__(GEMM_THREADS) gemm_kernel(const GTask* __restrict__ tasks,
                                                            const SnInfo* __restrict__ sn, double* panels,
                                                            const double* __restrict__ linv,
                                                            const long long* __restrict__ ucol_base,
                                                            const long long* __restrict__ ucol_map,
                                                            const int* __restrict__ posmap) {
  extern __shared__ __align__(16) double smem[];
  double* sA = smem;
  double* sB = smem + STAGES * BK * LDS;
  const GTask T = tasks[blockIdx.x];
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
  } else {
    A = panels + S.off + T.r0;
    B = panels + S.off + T.s0;
    lda = ldb = S.ld; arows = S.m - T.r0; brows = S.m - T.s0; K = S.k;
  }
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1, g = lane >> 2, t = lane & 3;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int nchunks = (K + BK - 1) / BK;
  auto load_chunk = [&](int chunk, int stage) {
    const int kc = chunk * BK;
    double* dA = sA + stage * BK * LDS;
    double* dB = sB + stage * BK * LDS;
#pragma unroll
    for (int i = 0; i < (BK * TILE / 2) / GEMM_THREADS; ++i) {
      const int p = tid + i * GEMM_THREADS;
      const int kk = p >> 5, rp = (p & 31) * 2;
      const bool kval = (kc + kk) < K;
      const int ra = kval ? max(0, min(2, arows - rp)) : 0;
      const int rb = kval ? max(0, min(2, brows - rp)) : 0;
      cp_async16(dA + kk * LDS + rp, ra ? A + (long long)(kc + kk) * lda + rp : A, ra * 8);
      cp_async16(dB + kk * LDS + rp, rb ? B + (long long)(kc + kk) * ldb + rp : B, rb * 8);
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
  // ---- epilogue: stage the 64x64 tile through shared memory (column-major, stride LDC), then
  // each warp streams whole 64-row columns: 16-byte vector RMW / stores (LOCAL, TRSM) or runs of
  // consecutive RED (SCATTER, relind runs are long: consecutive U rows land in consecutive
  // ancestor rows).  All destination loads of a thread are issued before its stores.
  constexpr int LDC = TILE + 4;   // 68 doubles: conflict-free fragment writes and v2 reads
  __syncthreads();
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
        if (gr < S.m && gr - S.k >= uc) atomicAdd(panels + cb + posmap[mb + gr], -sC[col * LDC + row]);
      }
    }
  }
}

// ----------------------------------------------------------------------------------------------
// potrf_kernel: one CTA (256 threads) factors the nb x nb (nb <= 64) diagonal block [c0, c0+nb) of
// supernode J ("DPOTRF") and forms X = L_bb^{-1} for TRSM-as-GEMM.
// The 64x64 lower triangle is cut into 4x4 register blocks; thread t < 136 owns block (bi, bj),
// bi >= bj.  Cholesky, right-looking, step j: the owners of column j publish it (double-buffered
// shared vector, ONE barrier per step), every thread scales its rows/columns by 1/sqrt(pivot) and
// applies the rank-1 update to its block.  Inverse, step s (forward substitution on I): the owners
// of row s of X scale it by 1/L_ss and publish it; rows r > s subtract L(r,s) X(s,:).
// The strict upper triangle of the panel is padding and is never written.  X is written to the
// task's workspace slot, column-major, ld 64, zero padded.  A pivot that is not > 0 (incl. NaN)
// records its global column (final numbering) with atomicMin (a7).
// ----------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(POTRF_THREADS) potrf_kernel(const PTask* __restrict__ tasks,
                                                              const SnInfo* __restrict__ sn,
                                                              const int* __restrict__ sfirst, double* panels,
                                                              double* linv, unsigned long long* fail) {
  __shared__ double vbuf[2][NBMAX];            // published column of L / row of X
  __shared__ double Ls[NBMAX][NBMAX + 1];      // Ls[row][col] = L(row, col) after the Cholesky
  __shared__ double invd[NBMAX];
  const PTask T = tasks[blockIdx.x];
  const SnInfo S = sn[T.sn];
  const int nb = T.nb, tid = threadIdx.x;
  // block coordinates: t -> (bi, bj), bi >= bj, row-major over the lower block triangle
  const bool owner = tid < 136;
  int bi = 0, bj = owner ? tid : 0;
  while (bj > bi) { bj -= bi + 1; ++bi; }
  const int r0 = 4 * bi, q0 = 4 * bj;
  double* P = panels + S.off + (long long)T.c0 * S.ld + T.c0;
  double a[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int r = r0 + i, c = q0 + q;
      a[i][q] = (owner && r < nb && c < nb && r >= c) ? P[(long long)c * S.ld + r] : 0.0;
    }
  int bad = -1;
  for (int jb = 0; jb < (nb + 3) / 4; ++jb) {
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      const int j = 4 * jb + jj;
      if (j >= nb) break;
      double* col = vbuf[j & 1];
      if (owner && bj == jb) {
#pragma unroll
        for (int i = 0; i < 4; ++i) col[r0 + i] = a[i][jj];
      }
      __syncthreads();
      const double d = col[j];
      const double l = sqrt(d), rl = 1.0 / l;
      if (bad < 0 && !(d > 0.0)) bad = j;
      double lr[4], lc[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        lr[i] = col[r0 + i] * rl;
        lc[i] = col[q0 + i] * rl;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (r0 + i >= q0 + q && q0 + q > j) a[i][q] -= lr[i] * lc[q];
      if (bj == jb) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int r = r0 + i;
          if (r > j) a[i][jj] = lr[i];
          else if (r == j) a[i][jj] = l;
        }
      }
      if (tid == 0) invd[j] = rl;
    }
  }
  if (tid == 0 && bad >= 0) atomicMin(fail, (unsigned long long)(sfirst[T.sn] + T.c0 + bad));
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int r = r0 + i, c = q0 + q;
      if (owner) Ls[r][c] = a[i][q];
      if (owner && r < nb && c < nb && r >= c) P[(long long)c * S.ld + r] = a[i][q];
    }
  // inverse: x = identity restricted to the block, forward substitution over pivot rows s
  double x[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int q = 0; q < 4; ++q) x[i][q] = (owner && r0 + i == q0 + q && r0 + i < nb) ? 1.0 : 0.0;
  __syncthreads();
  for (int sb = 0; sb < (nb + 3) / 4; ++sb) {
#pragma unroll
    for (int ss = 0; ss < 4; ++ss) {
      const int s = 4 * sb + ss;
      if (s >= nb) break;
      double* row = vbuf[s & 1];
      if (owner && bi == sb) {
        const double is = invd[s];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          x[ss][q] *= is;
          row[q0 + q] = x[ss][q];
        }
      }
      __syncthreads();
      if (owner && r0 + 3 > s) {
        double xs[4], lrs[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) xs[q] = row[q0 + q];
#pragma unroll
        for (int i = 0; i < 4; ++i) lrs[i] = Ls[r0 + i][s];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (r0 + i > s && q0 + q <= s) x[i][q] -= lrs[i] * xs[q];
      }
    }
  }
  double* W = linv + (long long)T.slot * (NBMAX * NBMAX);
  // the whole 64x64 slot is written: owners write their lower blocks, the rest writes zeros
  for (int e = tid; e < NBMAX * NBMAX; e += POTRF_THREADS) {
    const int c = e / NBMAX, r = e % NBMAX;
    if (r < c || r >= nb || c >= nb) W[e] = 0.0;
  }
  if (owner) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int r = r0 + i, c = q0 + q;
        if (r >= c && r < nb && c < nb) W[c * NBMAX + r] = x[i][q];
      }
  }
}

__global__ void init_scatter_kernel(const double* __restrict__ vals, const long long* __restrict__ amap,
                                    long long nnz, double* panels) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nnz; e += (long long)gridDim.x * blockDim.x)
    panels[amap[e]] = vals[e];
}

// Forward solve for the supernodes of one level: y_J := L_JJ^{-1} y_J, then y_R -= L_RJ y_J.
__global__ void solve_fwd_kernel(const int* __restrict__ sns, const SnInfo* __restrict__ sn,
                                 const int* __restrict__ sfirst, const long long* __restrict__ rows_ptr,
                                 const int* __restrict__ rows, const double* __restrict__ panels, double* y) {
  const int J = sns[blockIdx.x];
  const SnInfo S = sn[J];
  const int f = sfirst[J];
  const double* P = panels + S.off;
  for (int c = 0; c < S.k; ++c) {
    if (threadIdx.x == 0) y[f + c] /= P[(long long)c * S.ld + c];
    __syncthreads();
    const double xc = y[f + c];
    for (int r = c + 1 + threadIdx.x; r < S.k; r += blockDim.x) y[f + r] -= P[(long long)c * S.ld + r] * xc;
    __syncthreads();
  }
  const int* R = rows + rows_ptr[J];
  for (int r = S.k + threadIdx.x; r < S.m; r += blockDim.x) {
    double s = 0.0;
    for (int c = 0; c < S.k; ++c) s += P[(long long)c * S.ld + r] * y[f + c];
    atomicAdd(y + R[r], -s);
  }
}

// Backward solve for one level (root first): y_J := L_JJ^{-T} (y_J - L_RJ^T y_R).
__global__ void solve_bwd_kernel(const int* __restrict__ sns, const SnInfo* __restrict__ sn,
                                 const int* __restrict__ sfirst, const long long* __restrict__ rows_ptr,
                                 const int* __restrict__ rows, const double* __restrict__ panels, double* y) {
  const int J = sns[blockIdx.x];
  const SnInfo S = sn[J];
  const int f = sfirst[J];
  const double* P = panels + S.off;
  const int* R = rows + rows_ptr[J];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int c = warp; c < S.k; c += nw) {
    double s = 0.0;
    for (int r = S.k + lane; r < S.m; r += 32) s += P[(long long)c * S.ld + r] * y[R[r]];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) y[f + c] -= s;
  }
  __syncthreads();
  for (int c = S.k - 1; c >= 0; --c) {
    if (threadIdx.x == 0) y[f + c] /= P[(long long)c * S.ld + c];
    __syncthreads();
    const double xc = y[f + c];
    for (int r = threadIdx.x; r < c; r += blockDim.x) y[f + r] -= P[(long long)r * S.ld + c] * xc;
    __syncthreads();
  }
}

__global__ void permute_kernel(const int* __restrict__ perm, const double* __restrict__ in, double* out, long long n,
                               int inverse) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    if (inverse) out[i] = in[perm[i]];   // x[i] = z[pf[i]]
    else out[perm[i]] = in[i];           // y[pf[i]] = b[i]
  }
}

__global__ void gather_kernel(const double* __restrict__ src, const long long* __restrict__ idx, double* out, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = src[idx[i]];
}

// ---------------------------------------------------------------------------------------------- launchers
cudaError_t kernels_init_attributes() {
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(gemm_kernel<MODE_LOCAL>, cudaFuncAttributeMaxDynamicSharedMemorySize, GEMM_SMEM))) return e;
  if ((e = cudaFuncSetAttribute(gemm_kernel<MODE_TRSM>, cudaFuncAttributeMaxDynamicSharedMemorySize, GEMM_SMEM))) return e;
  if ((e = cudaFuncSetAttribute(gemm_kernel<MODE_SCATTER>, cudaFuncAttributeMaxDynamicSharedMemorySize, GEMM_SMEM))) return e;
  return cudaSuccess;
}

void launch_gemm(int mode, const GTask* tasks, int ntasks, const SnInfo* sn, double* panels, const double* linv,
                 const long long* ucol_base, const long long* ucol_map, const int* posmap, cudaStream_t st) {
  if (ntasks <= 0) return;
  if (mode == MODE_LOCAL)
    gemm_kernel<MODE_LOCAL><<<ntasks, GEMM_THREADS, GEMM_SMEM, st>>>(tasks, sn, panels, linv, ucol_base, ucol_map, posmap);
  else if (mode == MODE_TRSM)
    gemm_kernel<MODE_TRSM><<<ntasks, GEMM_THREADS, GEMM_SMEM, st>>>(tasks, sn, panels, linv, ucol_base, ucol_map, posmap);
  else
    gemm_kernel<MODE_SCATTER><<<ntasks, GEMM_THREADS, GEMM_SMEM, st>>>(tasks, sn, panels, linv, ucol_base, ucol_map, posmap);
}

void launch_potrf(const PTask* tasks, int ntasks, const SnInfo* sn, const int* sfirst, double* panels, double* linv,
                  unsigned long long* fail, cudaStream_t st) {
  if (ntasks <= 0) return;
  potrf_kernel<<<ntasks, POTRF_THREADS, 0, st>>>(tasks, sn, sfirst, panels, linv, fail);
}

void launch_init(const double* vals, const long long* amap, long long nnz, double* panels, cudaStream_t st) {
  if (nnz <= 0) return;
  long long blocks = (nnz + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  init_scatter_kernel<<<(int)blocks, 256, 0, st>>>(vals, amap, nnz, panels);
}

void launch_solve_fwd(const int* sns, int count, const SnInfo* sn, const int* sfirst, const long long* rows_ptr,
                      const int* rows, const double* panels, double* y, cudaStream_t st) {
  if (count > 0) solve_fwd_kernel<<<count, 256, 0, st>>>(sns, sn, sfirst, rows_ptr, rows, panels, y);
}
void launch_solve_bwd(const int* sns, int count, const SnInfo* sn, const int* sfirst, const long long* rows_ptr,
                      const int* rows, const double* panels, double* y, cudaStream_t st) {
  if (count > 0) solve_bwd_kernel<<<count, 256, 0, st>>>(sns, sn, sfirst, rows_ptr, rows, panels, y);
}
void launch_gather(const double* src, const long long* idx, double* out, long long n, cudaStream_t st) {
  if (n <= 0) return;
  long long blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  gather_kernel<<<(int)blocks, 256, 0, st>>>(src, idx, out, n);
}
void launch_permute(const int* perm, const double* in, double* out, long long n, int inverse, cudaStream_t st) {
  if (n <= 0) return;
  long long blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  permute_kernel<<<(int)blocks, 256, 0, st>>>(perm, in, out, n, inverse);
}

}  // namespace spchol
