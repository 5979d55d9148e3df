// DMMA issue model on one SM: cycles of 64 x 64 x 64 products from shared memory with 4 / 8 / 16
// warps resident in one CTA, and of the panel kernels' pk_mma (cp.async pipeline from L2) with K = 64
// and 256.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include
//   -I paper_2409_14009_b200/csrc tools/dmma_probe.cu -o tools/dmma_probe
#include "../paper_2409_14009_b200/csrc/kernels.cu"
#include <cstdio>
using namespace spchol;
__global__ void smem_mma(long long* out, double* sink, int reps) {
  extern __shared__ __align__(16) double sm[];
  for (int e = threadIdx.x; e < 2 * TILE * LDS; e += blockDim.x) sm[e] = 1e-3 * (e % 101);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = (warp >> 1) & 1, wn = warp & 1, g = lane >> 2, t = lane & 3;
  double acc[4][4][2] = {};
  const double* cA = sm + wm * 32 + g;
  const double* cB = sm + TILE * LDS + wn * 32 + g;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll 4
    for (int k = 0; k < TILE; k += 4) {
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
  }
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) s += acc[i][j][0] + acc[i][j][1];
  sink[threadIdx.x] = s;
  if (threadIdx.x == 0) out[0] = (t1 - t0) / reps;
}
template <int BKp, int STp>
__global__ void glob_mma(long long* out, double* M, int ld, int K, int reps) {
  extern __shared__ __align__(16) double sm[];
  double acc[4][4][2];
  long long tm = 0, ts = 0;
  for (int r = 0; r < reps; ++r) {
    long long t0 = clock64();
    pk_mma<BKp, STp>(M, ld, 64, M + 64, ld, 64, K, acc, sm);
    long long t1 = clock64();
    pk_store(acc, sm, M + 128 + (long long)K * ld, ld, 0, 64, 64, true, false);
    long long t2 = clock64();
    if (r > 0) { tm += t1 - t0; ts += t2 - t1; }
  }
  if (threadIdx.x == 0) { out[0] = tm / (reps - 1); out[1] = ts / (reps - 1); }
}
__global__ void dmma_lat(long long* out, double* sink, int n) {
  double acc[2] = {1e-3 * threadIdx.x, 0.0};
  const double a = 1.0000001, b = 0.9999999;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) dmma(acc, a, b);
  long long t1 = clock64();
  sink[threadIdx.x] = acc[0] + acc[1];
  if (threadIdx.x == 0) out[0] = (t1 - t0) / n;
}
int main() {
  long long* d; double* sink; double* M;
  cudaMalloc(&d, 64); cudaMalloc(&sink, 8192); cudaMalloc(&M, sizeof(double) * 256 * 600);
  cudaMemset(M, 0, sizeof(double) * 256 * 600);
  cudaFuncSetAttribute(smem_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, 80000);
  cudaFuncSetAttribute(glob_mma<8, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  cudaFuncSetAttribute(glob_mma<16, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  cudaFuncSetAttribute(glob_mma<16, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  cudaFuncSetAttribute(glob_mma<32, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  cudaFuncSetAttribute(glob_mma<8, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  dmma_lat<<<1, 32>>>(d, sink, 1000);
  { long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost); printf("dependent DMMA chain: %lld cycles per DMMA\n", h); }
  for (int warps : {4, 8, 16}) {
    smem_mma<<<1, 32 * warps, 2 * TILE * LDS * 8>>>(d, sink, 20);
    long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("smem 64^3 per warp-quad, %2d warps: %lld cycles per rep (%d DMMA per warp; %.1f FMA/clk/SM)\n", warps, h, 256,
           (double)warps * 256 * 256 / h);
  }
  for (int K : {64, 256}) {
    for (int v = 0; v < 5; ++v) {
      if (v == 0) glob_mma<8, 4><<<1, 128, 100000>>>(d, M, 256, K, 6);
      if (v == 1) glob_mma<16, 4><<<1, 128, 100000>>>(d, M, 256, K, 6);
      if (v == 2) glob_mma<16, 3><<<1, 128, 100000>>>(d, M, 256, K, 6);
      if (v == 3) glob_mma<32, 2><<<1, 128, 100000>>>(d, M, 256, K, 6);
      if (v == 4) glob_mma<8, 8><<<1, 128, 100000>>>(d, M, 256, K, 6);
      const char* nm[] = {"8x4", "16x4", "16x3", "32x2", "8x8"};
      long long h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
      printf("pk_mma %s K=%d: %lld cycles (%.1f FMA/clk), pk_store(sub): %lld cycles\n", nm[v], K, h[0], 64.0 * 64 * K / h[0], h[1]);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
