// FP64 peak microbenchmarks for B200 (sm_100a): DMMA (mma.sync m8n8k4 f64) and DFMA,
// plus a cuBLAS DGEMM as a measurement-only "achievable" reference (never on the product path),
// plus FP64 RED (atomicAdd) throughput for the relind scatter design.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu -lcublas
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
#include <cublas_v2.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while(0)

template <int CHAINS>
__global__ void dmma_loop(double* out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-9, b = seed * 0.5 + threadIdx.x * 1e-10;
  double c[CHAINS][2];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
__global__ void dfma_loop(double* out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-9, b = 1.0 - 1e-12;
  double c[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) c[i] = i * 1e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) c[i] = fma(c[i], b, a);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void red_random(double* buf, uint64_t nbuf, int per_thread, uint64_t seed) {
  uint64_t x = seed ^ (blockIdx.x * 1315423911ull + threadIdx.x * 2654435761ull);
  for (int i = 0; i < per_thread; ++i) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    atomicAdd(&buf[x % nbuf], 1.0);
  }
}
// runs: each warp writes 32 consecutive doubles (coalesced RED), random run start
__global__ void red_runs(double* buf, uint64_t nruns, int per_thread, uint64_t seed) {
  uint64_t x = seed ^ (blockIdx.x * 1315423911ull + (threadIdx.x >> 5) * 2654435761ull);
  for (int i = 0; i < per_thread; ++i) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    atomicAdd(&buf[(x % nruns) * 32 + (threadIdx.x & 31)], 1.0);
  }
}
__global__ void rmw_runs(double* buf, uint64_t nruns, int per_thread, uint64_t seed) {
  uint64_t x = seed ^ (blockIdx.x * 1315423911ull + (threadIdx.x >> 5) * 2654435761ull);
  for (int i = 0; i < per_thread; ++i) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    double* p = &buf[(x % nruns) * 32 + (threadIdx.x & 31)];
    *p = *p + 1.0;
  }
}

int main(int argc, char** argv) {
  int dev = 0; CK(cudaSetDevice(dev));
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, dev));
  int sms = prop.multiProcessorCount;
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  printf("{\"device\":\"%s\",\"sms\":%d,\"clock_khz_attr\":%d}\n", prop.name, sms, clk_khz);
  double* out; CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  // DMMA sweep: warps per SM
  for (int wps : {4, 8, 16}) {
    int threads = 32 * (wps > 8 ? 8 : wps);
    int blocks = sms * (wps > 8 ? wps / 8 : 1);
    int iters = 20000;
    dmma_loop<8><<<blocks, threads>>>(out, 100, 1.0);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); dmma_loop<8><<<blocks, threads>>>(out, iters, 1.0); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double flops = 2.0 * 256.0 * 8 * iters * (double)blocks * (threads / 32);
    printf("{\"kernel\":\"dmma_m8n8k4\",\"warps_per_sm\":%d,\"ms\":%.3f,\"tflops\":%.3f}\n", wps, best, flops / best / 1e9);
  }
  for (int wps : {8, 16, 32}) {
    int threads = 256; int blocks = sms * wps / 8; int iters = 20000;
    dfma_loop<8><<<blocks, threads>>>(out, 100, 1.0); CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); dfma_loop<8><<<blocks, threads>>>(out, iters, 1.0); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double flops = 2.0 * 8 * iters * (double)blocks * threads;
    printf("{\"kernel\":\"dfma\",\"warps_per_sm\":%d,\"ms\":%.3f,\"tflops\":%.3f}\n", wps, best, flops / best / 1e9);
  }
  // sustained DMMA: back to back ~4 s
  {
    int threads = 256, blocks = sms; int iters = 20000;
    cudaEventRecord(e0); int n = 0; float ms = 0;
    double flops1 = 2.0 * 256.0 * 8 * iters * (double)blocks * (threads / 32);
    while (true) {
      for (int k = 0; k < 20; ++k) dmma_loop<8><<<blocks, threads>>>(out, iters, 1.0);
      n += 20; cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      if (ms > 4000) break;
    }
    printf("{\"kernel\":\"dmma_m8n8k4_sustained\",\"seconds\":%.2f,\"tflops\":%.3f}\n", ms / 1e3, flops1 * n / ms / 1e9);
  }
  // cuBLAS DGEMM 8192^3 (measurement-only reference)
  {
    int N = 8192; size_t bytes = (size_t)N * N * 8; double *A, *B, *C;
    CK(cudaMalloc(&A, bytes)); CK(cudaMalloc(&B, bytes)); CK(cudaMalloc(&C, bytes));
    cudaMemset(A, 0, bytes); cudaMemset(B, 0, bytes); cudaMemset(C, 0, bytes);
    cublasHandle_t h; cublasCreate(&h); double al = 1.0, be = 0.0;
    cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_T, N, N, N, &al, A, N, B, N, &be, C, N); CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_T, N, N, N, &al, A, N, B, N, &be, C, N); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    printf("{\"kernel\":\"cublas_dgemm_8192\",\"ms\":%.3f,\"tflops\":%.3f}\n", best, 2.0 * N * (double)N * N / best / 1e9);
    // sustained cublas 4 s
    cudaEventRecord(e0); int n = 0; float ms = 0;
    while (true) { for (int k = 0; k < 5; ++k) cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_T, N, N, N, &al, A, N, B, N, &be, C, N);
      n += 5; cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1); if (ms > 4000) break; }
    printf("{\"kernel\":\"cublas_dgemm_8192_sustained\",\"seconds\":%.2f,\"tflops\":%.3f}\n", ms / 1e3, 2.0 * N * (double)N * N * n / ms / 1e9);
    cublasDestroy(h); cudaFree(A); cudaFree(B); cudaFree(C);
  }
  // FP64 RED throughput
  {
    uint64_t nbuf = (1ull << 30) / 8 * 2; double* buf; CK(cudaMalloc(&buf, nbuf * 8)); cudaMemset(buf, 0, nbuf * 8);
    int blocks = sms * 8, threads = 256, per = 256;
    red_random<<<blocks, threads>>>(buf, nbuf, 4, 1); CK(cudaDeviceSynchronize());
    float ms; cudaEventRecord(e0); red_random<<<blocks, threads>>>(buf, nbuf, per, 7); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double n = (double)blocks * threads * per;
    printf("{\"kernel\":\"red_f64_random\",\"ms\":%.3f,\"gops\":%.3f}\n", ms, n / ms / 1e6);
    cudaEventRecord(e0); red_runs<<<blocks, threads>>>(buf, nbuf / 32, per, 9); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"kernel\":\"red_f64_runs32\",\"ms\":%.3f,\"gops\":%.3f,\"gbs_rmw_equiv\":%.1f}\n", ms, n / ms / 1e6, n * 16 / ms / 1e6);
    cudaEventRecord(e0); rmw_runs<<<blocks, threads>>>(buf, nbuf / 32, per, 11); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"kernel\":\"rmw_f64_runs32\",\"ms\":%.3f,\"gops\":%.3f,\"gbs\":%.1f}\n", ms, n / ms / 1e6, n * 16 / ms / 1e6);
    cudaFree(buf);
  }
  return 0;
}
