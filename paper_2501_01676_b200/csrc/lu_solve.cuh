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
// X is n x NR row-major with row stride xstride(NR) (NR + 1 for NR > 1: the
// padding spreads the lanes of a warp over the shared-memory banks).
#pragma once
#include "common.cuh"

namespace bddc {
namespace lus {

constexpr int kP = 64;

template <int NR>
__host__ __device__ constexpr int xstride() { return NR == 1 ? 1 : NR + 1; }

// single right-hand side: warp per 4 rows (4 independent loads per lane in flight)
BDDC_DEV void rows_gemv1(const double* __restrict__ A, long long lda, int m, int k,
                         const double* X, double* Y, double alpha, double beta) {
  const int warp = (int)(threadIdx.x >> 5), lane = (int)(threadIdx.x & 31);
  const int nw = (int)(blockDim.x >> 5);
  for (int r0 = 4 * warp; r0 < m; r0 += 4 * nw) {
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    const double* a0 = A + (long long)r0 * lda;
    const int nr = min(4, m - r0);
    for (int c = lane; c < k; c += 32) {
      const double x = X[c];
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (i < nr) s[i] = fma(a0[(long long)i * lda + c], x, s[i]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s[i] += __shfl_xor_sync(0xffffffffu, s[i], o);
    if (lane < nr) {
      double t = s[0];
#pragma unroll
      for (int i = 1; i < 4; ++i)
        if (lane == i) t = s[i];
      Y[r0 + lane] = (beta == 0.0 ? 0.0 : beta * Y[r0 + lane]) + alpha * t;
    }
  }
}

// Y[r][q] = beta * Y[r][q] + alpha * sum_c A[r][c] X[c][q]   (r < m, c < k); warp per row
template <int NR>
BDDC_DEV void rows_gemv(const double* __restrict__ A, long long lda, int m, int k,
                        const double* X, double* Y, double alpha, double beta) {
  if (NR == 1) {
    rows_gemv1(A, lda, m, k, X, Y, alpha, beta);
    return;
  }
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
      for (int q = 0; q < NR; ++q) s[q] = fma(v, X[c * xstride<NR>() + q], s[q]);
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
      Y[r * xstride<NR>() + lane] = (beta == 0.0 ? 0.0 : beta * Y[r * xstride<NR>() + lane]) + alpha * t;
    }
  }
}

// Y[c][q] = beta * Y[c][q] + alpha * sum_r A[r][c] X[r][q]   (c < n, r < m); thread per column,
// the rows split over blockDim / n_cols groups and reduced through red (>= blockDim * NR doubles)
template <int NR>
BDDC_DEV void cols_acc(const double* __restrict__ A, long long lda, int r0, int m, int step, int c,
                       const double* X, double* s) {
  constexpr int XS = xstride<NR>();
  int r = r0;
  for (; r + 3 * step < m; r += 4 * step) {
    const double v0 = A[(long long)r * lda + c], v1 = A[(long long)(r + step) * lda + c];
    const double v2 = A[(long long)(r + 2 * step) * lda + c], v3 = A[(long long)(r + 3 * step) * lda + c];
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      s[q] = fma(v0, X[r * XS + q], s[q]);
      s[q] = fma(v1, X[(r + step) * XS + q], s[q]);
      s[q] = fma(v2, X[(r + 2 * step) * XS + q], s[q]);
      s[q] = fma(v3, X[(r + 3 * step) * XS + q], s[q]);
    }
  }
  for (; r < m; r += step) {
    const double v = A[(long long)r * lda + c];
#pragma unroll
    for (int q = 0; q < NR; ++q) s[q] = fma(v, X[r * XS + q], s[q]);
  }
}

template <int NR>
BDDC_DEV void cols_gemv(const double* __restrict__ A, long long lda, int m, int n,
                        const double* X, double* Y, double alpha, double beta, double* red) {
  constexpr int XS = xstride<NR>();
  const int nt = (int)blockDim.x;
  const int groups = max(1, nt / max(n, 1));
  const int grp = (int)threadIdx.x / max(n, 1), c = (int)threadIdx.x - grp * max(n, 1);
  if (n <= nt) {
    double s[NR];
#pragma unroll
    for (int q = 0; q < NR; ++q) s[q] = 0.0;
    if (grp < groups && c < n) cols_acc<NR>(A, lda, grp, m, groups, c, X, s);
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
        Y[c * XS + q] = (beta == 0.0 ? 0.0 : beta * Y[c * XS + q]) + alpha * s[q];
  } else {
    for (int cc = threadIdx.x; cc < n; cc += nt) {
      double s[NR];
#pragma unroll
      for (int q = 0; q < NR; ++q) s[q] = 0.0;
      cols_acc<NR>(A, lda, 0, m, 1, cc, X, s);
#pragma unroll
      for (int q = 0; q < NR; ++q)
        Y[cc * XS + q] = (beta == 0.0 ? 0.0 : beta * Y[cc * XS + q]) + alpha * s[q];
    }
  }
  __syncthreads();
}

// NR = 8 or 16 right-hand sides on the DMMA pipe (mma.sync m8n8k4.f64):
//   Y[r][q] = beta * Y[r][q] + alpha * sum_c op(A)[r][c] X[c][q]   (r < m, c < k, q < NR)
// op(A) = A (m x k, TA = false) or A^T (A stored k x m, TA = true).  A warp
// owns 8-row units (NR / 8 accumulators each, sharing the A fragment), up to
// four at a time, A fragments straight from global memory (32-byte row
// segments, every sector fully used) and X from shared memory: no shuffle
// reductions, unlike the warp-per-row products above.  Ends with a barrier.
template <int NR, bool TA>
BDDC_DEV void panel_mma(const double* __restrict__ A, long long lda, int m, int k,
                        const double* X, int xs, double* Y, int ys, double alpha, double beta) {
  constexpr int NB = NR / 8;
  const int warp = (int)(threadIdx.x >> 5), lane = (int)(threadIdx.x & 31);
  const int nw = (int)(blockDim.x >> 5);
  const int g = lane >> 2, t = lane & 3;
  const int mt = (m + 7) >> 3;  // 8-row units; a warp takes units warp, warp + nw, ... four at a time
  for (int u0 = warp; u0 < mt; u0 += 4 * nw) {
    int rr[4];
    bool on[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      on[i] = u0 + i * nw < mt;  // warp-uniform
      rr[i] = (u0 + i * nw) * 8 + g;
    }
    double acc[4][NB][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < NB; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll 4
    for (int p = 0; p < k; p += 4) {
      const int kk = p + t;
      const bool kin = kk < k;
      double bv[NB];
#pragma unroll
      for (int j = 0; j < NB; ++j) bv[j] = kin ? X[kk * xs + 8 * j + g] : 0.0;
      double a[4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
        a[i] = (kin && rr[i] < m) ? (TA ? A[(long long)kk * lda + rr[i]] : A[(long long)rr[i] * lda + kk])
                                  : 0.0;
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (on[i]) {
#pragma unroll
          for (int j = 0; j < NB; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], bv[j]);
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (rr[i] >= m) continue;
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        double* y = Y + rr[i] * ys + 8 * j + 2 * t;
#pragma unroll
        for (int h = 0; h < 2; ++h)
          y[h] = (beta == 0.0 ? 0.0 : beta * y[h]) + alpha * acc[i][j][h];
      }
    }
  }
  __syncthreads();
}

// L2 prefetch of an m x k block (row-major, ld doubles): one request per 128-byte
// line of every row, spread over the CTA.  The sweeps below request the block of
// the NEXT panel product while the current one runs (their loads are the kernel's
// stall: ~2/3 of the samples wait on a fragment coming from DRAM).
BDDC_DEV void prefetch_block_l2(const double* __restrict__ A, long long ld, int m, int k) {
  const int lines = (k * 8 + 127) >> 7;  // per row (rows are 16-byte aligned at best: +1 margin not needed)
  for (int idx = threadIdx.x; idx < m * lines; idx += blockDim.x) {
    const int r = idx / lines, l = idx - r * lines;
    asm volatile("prefetch.global.L2 [%0];\n" ::"l"(A + (long long)r * ld + l * 16));
  }
}

// x <- A^-1 x (TRANS: A^-T x); M: n x n LU (ld n) with P^-1 diagonal blocks;
// X: n rows of stride xstride(NR); tmp: 64 * xstride(NR) doubles; red: blockDim * NR
// doubles (transposed solve only)
template <int NR, bool TRANS>
BDDC_DEV void lu_solve(const double* __restrict__ M, int n, double* X, double* tmp, double* red) {
  constexpr int XS = xstride<NR>();
  const int np = (n + kP - 1) / kP;
  if constexpr (NR % 8 == 0) {
    // 8 or 16 right-hand sides: every panel product on the DMMA pipe
    if (!TRANS) {
      for (int j = 0; j < np; ++j) {
        const int j0 = j * kP, w = min(kP, n - j0), j1 = j0 + w;
        if (j1 < n) prefetch_block_l2(M + (long long)j1 * n + j0, n, n - j1, w);  // next product
        panel_mma<NR, false>(M + (long long)j0 * n + j0, n, w, w, X + j0 * XS, XS, tmp, XS, 1.0, 0.0);
        for (int i = threadIdx.x; i < w * XS; i += blockDim.x) X[j0 * XS + i] = tmp[i];
        __syncthreads();
        if (j1 < n) {
          if (j1 + kP <= n)  // the diagonal block after it
            prefetch_block_l2(M + (long long)j1 * n + j1, n, min(kP, n - j1), min(kP, n - j1));
          panel_mma<NR, false>(M + (long long)j1 * n + j0, n, n - j1, w, X + j0 * XS, XS, X + j1 * XS, XS,
                            -1.0, 1.0);
        }
      }
      for (int k = np - 2; k >= 0; --k) {
        const int k0 = k * kP, k1 = k0 + kP;
        if (k > 0) prefetch_block_l2(M + (long long)(k0 - kP) * n + k0, n, kP, n - k0);  // next
        panel_mma<NR, false>(M + (long long)k0 * n + k1, n, kP, n - k1, X + k1 * XS, XS, X + k0 * XS, XS,
                          -1.0, 1.0);
      }
    } else {
      for (int j = 0; j < np; ++j) {
        const int j0 = j * kP, w = min(kP, n - j0), j1 = j0 + w;
        if (j1 + kP < n)  // next product: pivot rows of the next panel, columns beyond it
          prefetch_block_l2(M + (long long)j1 * n + j1 + kP, n, min(kP, n - j1), n - j1 - kP);
        if (j1 < n)
          panel_mma<NR, true>(M + (long long)j0 * n + j1, n, n - j1, w, X + j0 * XS, XS, X + j1 * XS, XS,
                           -1.0, 1.0);
      }
      for (int k = np - 1; k >= 0; --k) {
        const int k0 = k * kP, w = min(kP, n - k0), k1 = k0 + w;
        if (k > 0)  // next product: the column panel of the previous pivot block below it
          prefetch_block_l2(M + (long long)k0 * n + k0 - kP, n, n - k0, kP);
        if (k1 < n)
          panel_mma<NR, true>(M + (long long)k1 * n + k0, n, w, n - k1, X + k1 * XS, XS, X + k0 * XS, XS,
                           -1.0, 1.0);
        panel_mma<NR, true>(M + (long long)k0 * n + k0, n, w, w, X + k0 * XS, XS, tmp, XS, 1.0, 0.0);
        for (int i = threadIdx.x; i < w * XS; i += blockDim.x) X[k0 * XS + i] = tmp[i];
        __syncthreads();
      }
    }
    return;
  }
  if (!TRANS) {
    for (int j = 0; j < np; ++j) {
      const int j0 = j * kP, w = min(kP, n - j0), j1 = j0 + w;
      rows_gemv<NR>(M + (long long)j0 * n + j0, n, w, w, X + j0 * XS, tmp, 1.0, 0.0);
      __syncthreads();
      for (int i = threadIdx.x; i < w * XS; i += blockDim.x) X[j0 * XS + i] = tmp[i];
      __syncthreads();
      if (j1 < n) rows_gemv<NR>(M + (long long)j1 * n + j0, n, n - j1, w, X + j0 * XS, X + j1 * XS, -1.0, 1.0);
      __syncthreads();
    }
    for (int k = np - 1; k >= 0; --k) {
      const int k0 = k * kP, w = min(kP, n - k0), k1 = k0 + w;
      if (k1 < n) rows_gemv<NR>(M + (long long)k0 * n + k1, n, w, n - k1, X + k1 * XS, X + k0 * XS, -1.0, 1.0);
      __syncthreads();
    }
  } else {
    for (int j = 0; j < np; ++j) {
      const int j0 = j * kP, w = min(kP, n - j0), j1 = j0 + w;
      if (j1 < n) cols_gemv<NR>(M + (long long)j0 * n + j1, n, w, n - j1, X + j0 * XS, X + j1 * XS, -1.0, 1.0, red);
    }
    for (int k = np - 1; k >= 0; --k) {
      const int k0 = k * kP, w = min(kP, n - k0), k1 = k0 + w;
      if (k1 < n) cols_gemv<NR>(M + (long long)k1 * n + k0, n, n - k1, w, X + k1 * XS, X + k0 * XS, -1.0, 1.0, red);
      // x_k = P_k^-T x_k
      cols_gemv<NR>(M + (long long)k0 * n + k0, n, w, w, X + k0 * XS, tmp, 1.0, 0.0, red);
      for (int i = threadIdx.x; i < w * XS; i += blockDim.x) X[k0 * XS + i] = tmp[i];
      __syncthreads();
    }
  }
}

}  // namespace lus
}  // namespace bddc
