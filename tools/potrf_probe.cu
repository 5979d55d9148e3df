// Microbenchmark / phase profile of the cdiv POTRF kernels on one 64x64 SPD block (one CTA, as on the
// critical chain).  Built standalone (the kernels' translation unit included), e.g.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DSPCHOL_P9_CLOCKS \
//        -I include -I paper_2409_14009_b200/csrc tools/potrf_probe.cu -o /tmp/potrf_probe
#include "../paper_2409_14009_b200/csrc/kernels.cu"
#include <cstdio>
#include <vector>
#include <cmath>
#include <algorithm>
using namespace spchol;
int main() {
  const int n = 64, ld = 64;
  std::vector<double> A(n * ld, 0.0);
  for (int j = 0; j < n; ++j)
    for (int i = j; i < n; ++i) A[j * ld + i] = i == j ? 2.0 * n : -1.0 / (1 + i + j);
  double *dA, *dW;
  SnInfo* dS;
  PTask* dT;
  int* dF;
  unsigned long long* dfail;
  cudaMalloc(&dA, sizeof(double) * n * ld);
  cudaMalloc(&dW, sizeof(double) * NBMAX * NBMAX);
  cudaMalloc(&dS, sizeof(SnInfo));
  cudaMalloc(&dT, sizeof(PTask));
  cudaMalloc(&dF, sizeof(int));
  cudaMalloc(&dfail, 8);
  SnInfo S{0, ld, n, n, -1};
  PTask T{0, 0, 64, 0};
  int f0 = 0;
  cudaMemcpy(dS, &S, sizeof(S), cudaMemcpyHostToDevice);
  cudaMemcpy(dT, &T, sizeof(T), cudaMemcpyHostToDevice);
  cudaMemcpy(dF, &f0, sizeof(int), cudaMemcpyHostToDevice);
  kernels_init_attributes();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  std::vector<double> L9(n * ld), W9(NBMAX * NBMAX), L10(n * ld), W10(NBMAX * NBMAX);
  for (int variant = 9; variant <= 10; ++variant) {
    float best = 1e9;
    for (int rep = 0; rep < 50; ++rep) {
      cudaMemcpy(dA, A.data(), sizeof(double) * n * ld, cudaMemcpyHostToDevice);
      cudaEventRecord(e0);
      if (variant == 9) potrf9_kernel<<<1, POTRF9_THREADS, POTRF9_SMEM>>>(dT, dS, dF, dA, dW, dfail);
      else potrf10_kernel<<<1, POTRF9_THREADS, POTRF10_SMEM>>>(dT, dS, dF, dA, dW, dfail);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    printf("potrf%d: best %.2f us (event, one CTA)\n", variant, best * 1e3);
    cudaMemcpy(variant == 9 ? L9.data() : L10.data(), dA, sizeof(double) * n * ld, cudaMemcpyDeviceToHost);
    cudaMemcpy(variant == 9 ? W9.data() : W10.data(), dW, sizeof(double) * NBMAX * NBMAX, cudaMemcpyDeviceToHost);
#ifdef SPCHOL_P9_CLOCKS
    if (variant == 9) {
      long long c[64];
      cudaMemcpyFromSymbol(c, p9_clocks, sizeof(c));
      for (int i = 1; i < 21 && c[i]; ++i) printf("  phase %2d: %lld cycles (cum %lld)\n", i, c[i] - c[i - 1], c[i] - c[0]);
    }
#endif
  }
  double dl = 0, dw = 0, ml = 0, mw = 0;
  for (int j = 0; j < n; ++j)
    for (int i = j; i < n; ++i) {
      dl = std::max(dl, std::fabs(L9[j * ld + i] - L10[j * ld + i]));
      ml = std::max(ml, std::fabs(L9[j * ld + i]));
    }
  for (int e = 0; e < NBMAX * NBMAX; ++e) {
    dw = std::max(dw, std::fabs(W9[e] - W10[e]));
    mw = std::max(mw, std::fabs(W9[e]));
  }
  printf("potrf10 vs potrf9: max|dL|/max|L| = %.3e, max|dX|/max|X| = %.3e\n", dl / ml, dw / mw);
  // partial block (nb = 40): padding path
  {
    PTask T2{0, 0, 40, 0};
    cudaMemcpy(dT, &T2, sizeof(T2), cudaMemcpyHostToDevice);
    for (int variant = 9; variant <= 10; ++variant) {
      cudaMemcpy(dA, A.data(), sizeof(double) * n * ld, cudaMemcpyHostToDevice);
      if (variant == 9) potrf9_kernel<<<1, POTRF9_THREADS, POTRF9_SMEM>>>(dT, dS, dF, dA, dW, dfail);
      else potrf10_kernel<<<1, POTRF9_THREADS, POTRF10_SMEM>>>(dT, dS, dF, dA, dW, dfail);
      cudaDeviceSynchronize();
      cudaMemcpy(variant == 9 ? L9.data() : L10.data(), dA, sizeof(double) * n * ld, cudaMemcpyDeviceToHost);
      cudaMemcpy(variant == 9 ? W9.data() : W10.data(), dW, sizeof(double) * NBMAX * NBMAX, cudaMemcpyDeviceToHost);
    }
    double d1 = 0, d2 = 0;
    for (int e = 0; e < n * ld; ++e) d1 = std::max(d1, std::fabs(L9[e] - L10[e]));
    for (int e = 0; e < NBMAX * NBMAX; ++e) d2 = std::max(d2, std::fabs(W9[e] - W10[e]));
    printf("nb=40: max|dL| = %.3e, max|dX| = %.3e\n", d1, d2);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
