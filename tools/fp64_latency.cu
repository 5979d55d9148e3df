// Latency microbenchmarks on B200: dependent DFMA / DMUL / rsqrt(double) / sqrt / div chains,
// __syncthreads with 5 warps, shared-memory store->barrier->load round trip.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double* out, long long* cyc, double x0, int n) {
  double x = x0 + threadIdx.x * 1e-9;
  __shared__ double s[256];
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, 0.999999, 1e-7);
  t1 = clock64(); if (threadIdx.x == 0) cyc[0] = (t1 - t0) / n;
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = x * 1.0000001;
  t1 = clock64(); if (threadIdx.x == 0) cyc[1] = (t1 - t0) / n;
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = rsqrt(x) + 0.5;
  t1 = clock64(); if (threadIdx.x == 0) cyc[2] = (t1 - t0) / n;
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = sqrt(x) + 0.5;
  t1 = clock64(); if (threadIdx.x == 0) cyc[3] = (t1 - t0) / n;
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = 1.0 / x + 0.5;
  t1 = clock64(); if (threadIdx.x == 0) cyc[4] = (t1 - t0) / n;
  t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  t1 = clock64(); if (threadIdx.x == 0) cyc[5] = (t1 - t0) / n;
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    s[(threadIdx.x + i) & 255] = x;
    __syncthreads();
    x = s[(threadIdx.x * 7 + i) & 255] + 1e-9;
  }
  t1 = clock64(); if (threadIdx.x == 0) cyc[6] = (t1 - t0) / n;
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) + 1e-9;
  t1 = clock64(); if (threadIdx.x == 0) cyc[7] = (t1 - t0) / n;
  out[threadIdx.x] = x;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 4096); cudaMallocManaged(&cyc, 64 * 8);
  for (int th : {32, 160}) {
    lat<<<1, th>>>(out, cyc, 1.5, 1000); cudaDeviceSynchronize();
    lat<<<1, th>>>(out, cyc, 1.5, 10000); cudaDeviceSynchronize();
    printf("threads %d: dfma %lld  dmul %lld  rsqrt %lld  sqrt %lld  div %lld  bar %lld  sts+bar+lds %lld  shfl %lld (cycles)\n",
           th, cyc[0], cyc[1], cyc[2], cyc[3], cyc[4], cyc[5], cyc[6], cyc[7]);
  }
  return 0;
}
