// Microbenchmark / phase profile of the cdiv POTRF kernels on one 64x64 SPD block (one CTA, as on the
// critical chain).  Built standalone (the kernels' translation unit included), e.g.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DSPCHOL_P9_CLOCKS \
//        -I include -I paper_2409_14009_b200/csrc tools/potrf_probe.cu -o /tmp/potrf_probe
#include "../paper_2409_14009_b200/csrc/kernels.cu"
#include <cstdio>
#include <vector>
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
  for (int variant = 9; variant <= 9; ++variant) {
    float best = 1e9;
    for (int rep = 0; rep < 50; ++rep) {
      cudaMemcpy(dA, A.data(), sizeof(double) * n * ld, cudaMemcpyHostToDevice);
      cudaEventRecord(e0);
      potrf9_kernel<<<1, POTRF9_THREADS, POTRF9_SMEM>>>(dT, dS, dF, dA, dW, dfail);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    printf("potrf%d: best %.2f us (event, one CTA)\n", variant, best * 1e3);
#ifdef SPCHOL_P9_CLOCKS
    if (variant == 9) {
      long long c[64];
      cudaMemcpyFromSymbol(c, p9_clocks, sizeof(c));
      for (int i = 1; i < 21 && c[i]; ++i) printf("  phase %2d: %lld cycles (cum %lld)\n", i, c[i] - c[i - 1], c[i] - c[0]);
      for (int p = 0; p < 7; ++p)
        printf("  panel %d phase-2 start %lld: t0 tile done +%lld, t0 diag done +%lld, t64 X_p done +%lld, t32 syrk done +%lld, t64 syrk done +%lld, barrier +%lld\n",
               p, c[3 + 2 * p] - c[0], c[21 + p] - c[3 + 2 * p], c[29 + p] - c[3 + 2 * p], c[37 + p] - c[3 + 2 * p],
               c[45 + p] - c[3 + 2 * p], c[53 + p] - c[3 + 2 * p], c[4 + 2 * p] - c[3 + 2 * p]);
    }
#endif
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
