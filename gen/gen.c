/*
 * Seeded synthetic input generators shared by the oracle tests and the CUDA path.
 * This module holds NONE of the factorization's arithmetic: it only builds inputs
 * (SURVEY.md §8(d) "Generator", App. A (1)).
 *
 *   - grid stencil matrices (2D 5/9-point, 3D 7/27-point, 3-dof 27-point "elasticity-like"
 *     K27 (x) B with B = [[3,1,1],[1,3,1],[1,1,3]]), lower-triangle CSC, ORIGINAL numbering,
 *     rows strictly increasing, diagonal first (the C-ABI input contract);
 *   - geometric nested-dissection permutation (old -> new), the `perm` handed to analyze
 *     (stands in for METIS, §4.1);
 *   - splitmix64 stream and the right-hand side b = A x*, x*_i ~ U[-1,1).
 *   - lower-CSC symmetric mat-vec (y = A x) used only to build b and to measure residuals.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---- splitmix64 ---- */
uint64_t gen_splitmix64_next(uint64_t* state) {
  uint64_t z = (*state += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
/* uniform in [0,1) with 53 random bits */
static double u01(uint64_t* s) { return (double)(gen_splitmix64_next(s) >> 11) * (1.0 / 9007199254740992.0); }

void gen_uniform(uint64_t seed, int64_t n, double lo, double hi, double* out) {
  uint64_t s = seed;
  for (int64_t i = 0; i < n; ++i) out[i] = lo + (hi - lo) * u01(&s);
}

/* ---- stencils ---- kind: 5 (2D 5-pt), 9 (2D 9-pt), 7 (3D 7-pt), 27 (3D 27-pt). dof 1 or 3. */
static int in_stencil(int kind, int dx, int dy, int dz) {
  int ax = abs(dx), ay = abs(dy), az = abs(dz);
  if (ax > 1 || ay > 1 || az > 1) return 0;
  switch (kind) {
    case 5: return az == 0 && ax + ay == 1;
    case 9: return az == 0 && ax + ay >= 1;
    case 7: return ax + ay + az == 1;
    case 27: return ax + ay + az >= 1;
  }
  return 0;
}
static double stencil_diag(int kind) { return kind == 5 ? 4.0 : kind == 9 ? 8.0 : kind == 7 ? 6.0 : 26.0; }
static const double B3[3][3] = {{3, 1, 1}, {1, 3, 1}, {1, 1, 3}};

/* Count (values==NULL) or fill the lower CSC. colptr has n+1 entries. Returns nnz(lower). */
int64_t gen_grid_csc(int kind, int kx, int ky, int kz, int dof,
                     int64_t* colptr, int32_t* rowidx, double* values) {
  int64_t nn = (int64_t)kx * ky * kz, n = nn * dof, p = 0;
  for (int64_t node = 0; node < nn; ++node) {
    int x = (int)(node % kx), y = (int)((node / kx) % ky), z = (int)(node / ((int64_t)kx * ky));
    for (int d = 0; d < dof; ++d) {
      int64_t col = node * dof + d;
      if (colptr) colptr[col] = p;
      for (int dz = -1; dz <= 1; ++dz)
        for (int dy = -1; dy <= 1; ++dy)
          for (int dx = -1; dx <= 1; ++dx) {
            int self = (dx == 0 && dy == 0 && dz == 0);
            if (!self && !in_stencil(kind, dx, dy, dz)) continue;
            int X = x + dx, Y = y + dy, Z = z + dz;
            if (X < 0 || Y < 0 || Z < 0 || X >= kx || Y >= ky || Z >= kz) continue;
            int64_t q = ((int64_t)Z * ky + Y) * kx + X;
            double kv = self ? stencil_diag(kind) : -1.0;
            for (int e = 0; e < dof; ++e) {
              int64_t row = q * dof + e;
              if (row < col) continue;
              if (rowidx) rowidx[p] = (int32_t)row;
              if (values) values[p] = dof == 1 ? kv : kv * B3[d][e];
              ++p;
            }
          }
    }
  }
  if (colptr) colptr[n] = p;
  return p;
}

/* ---- geometric nested dissection ---- */
typedef struct { int kx, ky, kz; int64_t next; int32_t* order; } nd_ctx;
static void emit(nd_ctx* c, int x, int y, int z) { c->order[c->next++] = (int32_t)(((int64_t)z * c->ky + y) * c->kx + x); }
static void nd(nd_ctx* c, int x0, int x1, int y0, int y1, int z0, int z1) {
  int lx = x1 - x0, ly = y1 - y0, lz = z1 - z0;
  if (lx <= 0 || ly <= 0 || lz <= 0) return;
  if (lx == 1 && ly == 1 && lz == 1) { emit(c, x0, y0, z0); return; }
  int axis = 0, len = lx;            /* longest axis, ties x < y < z */
  if (ly > len) { axis = 1; len = ly; }
  if (lz > len) { axis = 2; len = lz; }
  if (axis == 0) {
    int m = x0 + lx / 2;
    nd(c, x0, m, y0, y1, z0, z1); nd(c, m + 1, x1, y0, y1, z0, z1);
    for (int z = z0; z < z1; ++z) for (int y = y0; y < y1; ++y) emit(c, m, y, z);
  } else if (axis == 1) {
    int m = y0 + ly / 2;
    nd(c, x0, x1, y0, m, z0, z1); nd(c, x0, x1, m + 1, y1, z0, z1);
    for (int z = z0; z < z1; ++z) for (int x = x0; x < x1; ++x) emit(c, x, m, z);
  } else {
    int m = z0 + lz / 2;
    nd(c, x0, x1, y0, y1, z0, m); nd(c, x0, x1, y0, y1, m + 1, z1);
    for (int y = y0; y < y1; ++y) for (int x = x0; x < x1; ++x) emit(c, x, y, m);
  }
}
/* perm[old] = new, over n = kx*ky*kz*dof unknowns; dofs of a node stay consecutive. */
int gen_nd_perm(int kx, int ky, int kz, int dof, int32_t* perm) {
  int64_t nn = (int64_t)kx * ky * kz;
  int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nn > 0 ? nn : 1));
  if (!order) return -1;
  nd_ctx c = {kx, ky, kz, 0, order};
  nd(&c, 0, kx, 0, ky, 0, kz);
  if (c.next != nn) { free(order); return -2; }
  for (int64_t pos = 0; pos < nn; ++pos)
    for (int d = 0; d < dof; ++d) perm[(int64_t)order[pos] * dof + d] = (int32_t)(pos * dof + d);
  free(order);
  return 0;
}

/* y = A x with A = lower + lower^T - diag (lower CSC). */
void gen_symv_lower(int64_t n, const int64_t* colptr, const int32_t* rowidx, const double* values,
                    const double* x, double* y) {
  memset(y, 0, sizeof(double) * (size_t)n);
  for (int64_t j = 0; j < n; ++j)
    for (int64_t p = colptr[j]; p < colptr[j + 1]; ++p) {
      int64_t i = rowidx[p];
      y[i] += values[p] * x[j];
      if (i != j) y[j] += values[p] * x[i];
    }
}
