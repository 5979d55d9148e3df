#include "/root/repo/paper_2409_14009_b200/csrc/kernels.cu"
#include <cstdio>
using namespace spchol;
__global__ void tile_k(long long* out, int nlanes, int variant) {
  extern __shared__ __align__(16) double sm[];
  for (int e = threadIdx.x; e < NBMAX * P9_LD * 2; e += blockDim.x) sm[e] = 0.001 * (e % 97);
  __syncthreads();
  long long t0 = clock64();
  if (threadIdx.x < nlanes) {
    if (variant == 0) p9_syrk_tile(sm, 0, 8 + 4 * (threadIdx.x % 3), 8);
    else {
      int bad = -1;
      p9_diag<true>(sm, sm + NBMAX * P9_LD, 8, 64, bad, 0);
    }
  }
  __syncwarp();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = t1 - t0;
}
int main() {
  long long* d; cudaMalloc(&d, 8);
  cudaFuncSetAttribute(tile_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 80000);
  for (int v = 0; v < 2; ++v)
    for (int nl : {1, 3, 32}) {
      long long best = 1 << 30;
      for (int r = 0; r < 20; ++r) {
        tile_k<<<1, 32, 80000>>>(d, nl, v);
        long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        if (h < best) best = h;
      }
      printf("%s lanes=%d: %lld cycles\n", v == 0 ? "syrk tile" : "diag 8x8 + update", nl, best);
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
