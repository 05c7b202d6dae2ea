// Batched solves with the blocked no-pivot LU of schur_eliminate (64-wide
// panels, "rows below only" form), one CTA per matrix, right-hand sides in
// shared memory:
//   A = Lt U,  Lt block lower with diagonal blocks P_k and A21^(k) below
//   (the column panels as they were when panel k was eliminated), U unit
//   block upper with W_k = P_k^-1 A12^(k) in the pivot rows.  The diagonal
//   blocks hold P_k^-1 (lu_diag_pinv_kernel), so every matrix element is read
//   exactly once per solve.
//   A x = b :  for k up:   x_k = P_k^-1 x_k ; x_(>k) -= A21^(k) x_k
//              for k down: x_k -= W_k x_(>k)
//   A^T x = b: for k up:   x_(>k) -= W_k^T x_k
//              for k down: x_k = P_k^-T (x_k - A21^(k)T x_(>k))
// X is n x NR row-major (X[r * NR + q]).
#pragma once
#include "common.cuh"

namespace bddc {
namespace lus {

constexpr int kP = 64;

// Y[r][q] = beta * Y[r][q] + alpha * sum_c A[r][c] X[c][q]   (r < m, c < k); warp per row
template <int NR>
BDDC_DEV void rows_gemv(const double* __restrict__ A, long long lda, int m, int k,
                        const double* X, double* Y, double alpha, double beta) {
  const int warp = (int)(threadIdx.x >> 5), lane = (int)(threadIdx.x & 31);
  const int nw = (int)(blockDim.x >> 5);
  for (int r = warp; r < m; r += nw) {
    const double* a = A + (long long)r * lda;
    double s[NR];
#pragma unroll
    for (int q = 0; q < NR; ++q) s[q] = 0.0;
    for (int c = lane; c < k; c += 32) {
      const double v = a[c];
#pragma unroll
      for (int q = 0; q < NR; ++q) s[q] = fma(v, X[c * NR + q], s[q]);
    }
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      double t = s[q];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      s[q] = t;
    }
    if (lane < NR) {
      double t = 0.0;
#pragma unroll
      for (int q = 0; q < NR; ++q)
        if (q == lane) t = s[q];
      Y[r * NR + lane] = (beta == 0.0 ? 0.0 : beta * Y[r * NR + lane]) + alpha * t;
    }
  }
}

// Y[c][q] = beta * Y[c][q] + alpha * sum_r A[r][c] X[r][q]   (c < n, r < m); thread per column,
// the rows split over blockDim / n_cols groups and reduced through red (>= blockDim * NR doubles)
template <int NR>
BDDC_DEV void cols_gemv(const double* __restrict__ A, long long lda, int m, int n,
                        const double* X, double* Y, double alpha, double beta, double* red) {
  const int nt = (int)blockDim.x;
  const int groups = max(1, nt / max(n, 1));
  const int grp = (int)threadIdx.x / max(n, 1), c = (int)threadIdx.x - grp * max(n, 1);
  if (n <= nt) {
    double s[NR];
#pragma unroll
    for (int q = 0; q < NR; ++q) s[q] = 0.0;
    if (grp < groups && c < n) {
      for (int r = grp; r < m; r += groups) {
        const double v = A[(long long)r * lda + c];
#pragma unroll
        for (int q = 0; q < NR; ++q) s[q] = fma(v, X[r * NR + q], s[q]);
      }
    }
    if (groups > 1) {
      if (grp < groups && c < n)
#pragma unroll
        for (int q = 0; q < NR; ++q) red[(grp * n + c) * NR + q] = s[q];
      __syncthreads();
      if (grp == 0 && c < n) {
        for (int g2 = 1; g2 < groups; ++g2)
#pragma unroll
          for (int q = 0; q < NR; ++q) s[q] += red[(g2 * n + c) * NR + q];
      }
    }
    if (grp == 0 && c < n)
#pragma unroll
      for (int q = 0; q < NR; ++q)
        Y[c * NR + q] = (beta == 0.0 ? 0.0 : beta * Y[c * NR + q]) + alpha * s[q];
  } else {
    for (int cc = threadIdx.x; cc < n; cc += nt) {
      double s[NR];
#pragma unroll
      for (int q = 0; q < NR; ++q) s[q] = 0.0;
      for (int r = 0; r < m; ++r) {
        const double v = A[(long long)r * lda + cc];
#pragma unroll
        for (int q = 0; q < NR; ++q) s[q] = fma(v, X[r * NR + q], s[q]);
      }
#pragma unroll
      for (int q = 0; q < NR; ++q)
        Y[cc * NR + q] = (beta == 0.0 ? 0.0 : beta * Y[cc * NR + q]) + alpha * s[q];
    }
  }
  __syncthreads();
}

// x <- A^-1 x (TRANS: A^-T x); M: n x n LU (ld n) with P^-1 diagonal blocks;
// tmp: 64 * NR doubles; red: blockDim * NR doubles (transposed solve only)
template <int NR, bool TRANS>
BDDC_DEV void lu_solve(const double* __restrict__ M, int n, double* X, double* tmp, double* red) {
  const int np = (n + kP - 1) / kP;
  if (!TRANS) {
    for (int j = 0; j < np; ++j) {
      const int j0 = j * kP, w = min(kP, n - j0), j1 = j0 + w;
      rows_gemv<NR>(M + (long long)j0 * n + j0, n, w, w, X + j0 * NR, tmp, 1.0, 0.0);
      __syncthreads();
      for (int i = threadIdx.x; i < w * NR; i += blockDim.x) X[j0 * NR + i] = tmp[i];
      __syncthreads();
      if (j1 < n) rows_gemv<NR>(M + (long long)j1 * n + j0, n, n - j1, w, X + j0 * NR, X + j1 * NR, -1.0, 1.0);
      __syncthreads();
    }
    for (int k = np - 1; k >= 0; --k) {
      const int k0 = k * kP, w = min(kP, n - k0), k1 = k0 + w;
      if (k1 < n) rows_gemv<NR>(M + (long long)k0 * n + k1, n, w, n - k1, X + k1 * NR, X + k0 * NR, -1.0, 1.0);
      __syncthreads();
    }
  } else {
    for (int j = 0; j < np; ++j) {
      const int j0 = j * kP, w = min(kP, n - j0), j1 = j0 + w;
      if (j1 < n) cols_gemv<NR>(M + (long long)j0 * n + j1, n, w, n - j1, X + j0 * NR, X + j1 * NR, -1.0, 1.0, red);
    }
    for (int k = np - 1; k >= 0; --k) {
      const int k0 = k * kP, w = min(kP, n - k0), k1 = k0 + w;
      if (k1 < n) cols_gemv<NR>(M + (long long)k1 * n + k0, n, n - k1, w, X + k1 * NR, X + k0 * NR, -1.0, 1.0, red);
      // x_k = P_k^-T x_k
      cols_gemv<NR>(M + (long long)k0 * n + k0, n, w, w, X + k0 * NR, tmp, 1.0, 0.0, red);
      for (int i = threadIdx.x; i < w * NR; i += blockDim.x) X[k0 * NR + i] = tmp[i];
      __syncthreads();
    }
  }
}

}  // namespace lus
}  // namespace bddc
