// Timeline of the fused outer-block cdiv (panel_diag_kernel + panel_below_kernel) on a dense SPD
// matrix held as one supernode: globaltimer stamps per task (SPCHOL_PK_CLOCKS).  Built standalone:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DSPCHOL_PK_CLOCKS -DSPCHOL_P9_CLOCKS \
//        -I include -I paper_2409_14009_b200/csrc tools/panel_probe.cu -o /tmp/panel_probe
#include "../paper_2409_14009_b200/csrc/kernels.cu"
#include <cstdio>
#include <vector>
using namespace spchol;
int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 2048, ld = n, W = 256;
  std::vector<double> A((size_t)n * ld, 0.0);
  for (int j = 0; j < n; ++j)
    for (int i = j; i < n; ++i) A[(size_t)j * ld + i] = i == j ? 2.0 * n : -1.0 / (1 + i + j);
  double *dA, *dX;
  SnInfo* dS;
  PanTask* dT;
  int *dsf, *dsync;
  unsigned long long* dfail;
  cudaMalloc(&dA, sizeof(double) * (size_t)n * ld);
  cudaMalloc(&dX, sizeof(double) * NBMAX * NBMAX * (n / 64 + 1));
  cudaMalloc(&dS, sizeof(SnInfo));
  cudaMalloc(&dT, sizeof(PanTask) * 4096);
  cudaMalloc(&dsf, sizeof(int) * 2);
  cudaMalloc(&dsync, sizeof(int) * 4096);
  cudaMalloc(&dfail, 8);
  SnInfo S{0, ld, n, n, -1};
  cudaMemcpy(dS, &S, sizeof(S), cudaMemcpyHostToDevice);
  cudaMemset(dsf, 0, 8);
  kernels_init_attributes();
  cudaStream_t st;
  cudaStreamCreate(&st);
  for (int C = 0; C < 2; ++C) {
    const int c0 = C * W, w = W, nbk = 4, ntile = (n - c0 + 63) / 64, pw = C ? W : 0;
    std::vector<PanTask> t;
    for (int q = 0; pw > 0 && q < 4; ++q)
      for (int i = 0; i < nbk; ++i)
        for (int j = 0; j <= i; ++j) t.push_back(PanTask{0, c0, w, i, j, C * 4, 0, pw, q});
    for (int i = 0; i < nbk; ++i)
      for (int j = 0; j <= i; ++j) t.push_back(PanTask{0, c0, w, i, j, C * 4, 0, pw, -1});
    const int nd = (int)t.size();
    for (int j = 0; j < nbk; ++j)
      for (int i = nbk; i < ntile; ++i) t.push_back(PanTask{0, c0, w, i, j, C * 4, 0, pw, -1});
    cudaMemcpy(dT, t.data(), sizeof(PanTask) * t.size(), cudaMemcpyHostToDevice);
    float best = 1e9;
    for (int rep = 0; rep < 20; ++rep) {
      cudaMemcpy(dA, A.data(), sizeof(double) * (size_t)n * ld, cudaMemcpyHostToDevice);
      cudaMemset(dsync, 0, sizeof(int) * 4096);
      cudaMemset(dfail, 0xFF, 8);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0, st);
      launch_panel(dT, nd, (int)t.size() - nd, dsync + 4000, dsync, dS, dsf, dA, dX, dfail, 0, st, -1, 4000, n / 64 + 1);
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    long long c[8192][8];
    cudaMemcpyFromSymbol(c, pk_clk, sizeof(c));
    long long t0 = c[0][0];
    for (int q = 0; q < nd; ++q) t0 = std::min(t0, c[q][0]);
    printf("outer block %d (pw %d): best %.1f us; diag-region tasks (ns from first claim):\n", C, pw, best * 1e3);
    for (int q = 0; q < nd; ++q) {
      if (t[q].q >= 0) continue;
      printf("  (%d,%d) claim %6lld next %6lld", t[q].tile, t[q].blk, c[q][0] - t0, c[q][1] - t0);
      if (t[q].blk == t[q].tile)
        printf(" steps %6lld waited %6lld L-pub %6lld syrk %6lld potrf-done %6lld", c[q][2] - t0, c[q][3] - t0,
               c[q][4] - t0, c[q][5] - t0, c[q][6] - t0);
      else
        printf(" done %6lld", c[q][7] - t0);
      printf("\n");
    }
    long long bmax = 0;
    for (int q = 0; q < (int)t.size() - nd; ++q) bmax = std::max(bmax, c[4096 + q][2] - t0);
    printf("  below blocks %d: first claim %lld, first next-done %lld, last done %lld\n", (int)t.size() - nd,
           c[4096][0] - t0, c[4096][1] - t0, bmax);
  }
  long long p9[64];
  cudaMemcpyFromSymbol(p9, p9_clocks, sizeof(p9));
  printf("last potrf9 phases (cycles):");
  for (int i = 1; i < 21 && p9[i]; ++i) printf(" %lld", p9[i] - p9[i - 1]);
  printf("\n%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
