// Register-resident block Gauss-Jordan inverse of one <= 64 x 64 matrix per
// 256-thread CTA (the pivot-block inverse of the blocked eliminations and the
// per-slot glob Schur blocks).
#pragma once
#include "common.cuh"
#include "tile_mma.cuh"

namespace bddc {

struct RegGjSmem {
  double rowb[2][4][kTile];
  double colb[2][4][kTile];
  int bad;
};

// Inverse of the w x w (w <= 64) matrix M (leading dimension L) by
// Gauss-Jordan without pivoting, written to out (leading dimension ldo).
// Needs blockDim.x == 256.  Returns true (in every thread) when a pivot is
// zero / non-finite, or <= 0 with require_positive (the LDL^T pivots: the
// cho_factor criterion).  piv: the w scalar pivots (may be null).
BDDC_DEV bool reg_gj64(const double* __restrict__ M, long long L, int w, double* __restrict__ out,
                       long long ldo, int require_positive, double* __restrict__ piv,
                       RegGjSmem& sm) {
  // Register-resident block Gauss-Jordan with 4x4 pivot blocks: thread t owns
  // column c = t % 64 and rows r0 + 4 j (r0 = t / 64, j < 16), so the four
  // rows of a pivot block are rows of the four thread groups.  The pivot rows
  // and columns of step s go through double-buffered shared memory and are
  // published while step s-1 updates them: one barrier per 4 pivots.
  // Scalar pivots (the LU diagonal) come out of the 4x4 inversions.
  auto& rowb = sm.rowb;
  auto& colb = sm.colb;
  int& bad = sm.bad;
  const int c = threadIdx.x & 63, r0 = threadIdx.x >> 6;
  double a[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int r = r0 + 4 * j;
    a[j] = (r < w && c < w) ? M[(long long)r * L + c] : (r == c ? 1.0 : 0.0);
    if (j == 0) rowb[0][r0][c] = a[j];
    if (c < 4) colb[0][c][r] = a[j];
  }
  if (threadIdx.x == 0) bad = 0;
  const int nsteps = (w + 3) >> 2;
  for (int s = 0; s < nsteps; ++s) {
    const int par = s & 1, p = 4 * s;
    __syncthreads();
    // 4x4 pivot block and its inverse (every thread, in registers)
    double Mi[4][4], dpiv[4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) Mi[i][jj] = rowb[par][i][p + jj];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double pv = Mi[q][q];
      dpiv[q] = pv;
      const double ip = 1.0 / pv;
      double rowq[4], colq[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        rowq[x] = Mi[q][x];
        colq[x] = Mi[x][q];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          if (i == q) Mi[i][jj] = (jj == q) ? ip : rowq[jj] * ip;
          else Mi[i][jj] = (jj == q) ? -colq[i] * ip : Mi[i][jj] - colq[i] * rowq[jj] * ip;
        }
    }
    if (threadIdx.x == 0) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (p + q >= w) break;
        const double pv = dpiv[q];
        if (piv) piv[p + q] = pv;
        if (!(pv == pv) || pv == 0.0 || isinf(pv) || (require_positive && !(pv > 0.0))) bad = 1;
      }
    }
    // u = Mi * (pivot rows at column c)
    double u[4];
    {
      double rb[4];
#pragma unroll
      for (int l = 0; l < 4; ++l) rb[l] = rowb[par][l][c];
#pragma unroll
      for (int i = 0; i < 4; ++i) u[i] = Mi[i][0] * rb[0] + Mi[i][1] * rb[1] + Mi[i][2] * rb[2] + Mi[i][3] * rb[3];
    }
    const bool cpiv = (c >= p) && (c < p + 4);
    const int jc = c - p;
    double mcol[4];  // Mi[:, jc] when c is a pivot column
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      double v = 0.0;
#pragma unroll
      for (int jj = 0; jj < 4; ++jj)
        if (jj == jc) v = Mi[l][jj];
      mcol[l] = v;
    }
    const int nx = p + 4;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int r = r0 + 4 * j;
      double v;
      if (j == s) {  // pivot row p + r0
        // row r0 of Mi (pivot block) or row r0 of Mi * rowb
        double mrow = 0.0, urow = 0.0;
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (i == r0) {
            urow = u[i];
#pragma unroll
            for (int jj = 0; jj < 4; ++jj)
              if (jj == jc) mrow = Mi[i][jj];
          }
        v = cpiv ? mrow : urow;
      } else {
        const double f0 = colb[par][0][r], f1 = colb[par][1][r], f2 = colb[par][2][r],
                     f3 = colb[par][3][r];
        v = cpiv ? -(f0 * mcol[0] + f1 * mcol[1] + f2 * mcol[2] + f3 * mcol[3])
                 : a[j] - (f0 * u[0] + f1 * u[1] + f2 * u[2] + f3 * u[3]);
      }
      a[j] = v;
      if (j == s + 1) rowb[par ^ 1][r0][c] = v;
      if (c >= nx && c < nx + 4) colb[par ^ 1][c - nx][r] = v;
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int r = r0 + 4 * j;
    if (r < w && c < w) out[r * ldo + c] = a[j];
  }
  const bool failed = bad != 0;
  __syncthreads();  // sm reusable after return
  return failed;
}


}  // namespace bddc
