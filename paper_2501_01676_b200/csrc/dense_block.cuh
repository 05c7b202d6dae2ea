// CTA-cooperative small dense linear algebra in fp64 (row-major, any
// leading dimension, generic pointers: shared or global memory).
//
// Every routine must be called by all threads of the block with uniform
// arguments; each ends with __syncthreads() so results are visible.
// These are the per-glob building blocks of the face / edge eigenproblems
// (reference linalg.py, substructuring.py:161-171, scaling.py:10-25,
// adaptive.py:57-206).
#pragma once
#include "common.cuh"

namespace bddc {
namespace blk {

BDDC_DEV int tid() { return threadIdx.x; }
BDDC_DEV int nth() { return blockDim.x; }

// row-major 2D iteration without integer division: warp w takes rows
// w, w + nwarps, ...; lanes stride the columns.
#define BLK_FOR_RC(M, N)                                                   \
  for (int r = (int)(threadIdx.x >> 5); r < (M); r += (int)(blockDim.x >> 5)) \
    for (int c = (int)(threadIdx.x & 31); c < (N); c += 32)

BDDC_DEV void copy(double* dst, int ldd, const double* src, int lds, int m, int n) {
  BLK_FOR_RC(m, n) dst[r * ldd + c] = src[r * lds + c];
  __syncthreads();
}

BDDC_DEV void set_identity(double* A, int ld, int m, int n) {
  BLK_FOR_RC(m, n) A[r * ld + c] = (r == c) ? 1.0 : 0.0;
  __syncthreads();
}

BDDC_DEV void fill(double* A, int ld, int m, int n, double v) {
  BLK_FOR_RC(m, n) A[r * ld + c] = v;
  __syncthreads();
}

// L2 prefetch of `count` contiguous doubles (every 128-byte line once, whole
// block): the cold operand blocks of a glob kernel are requested up front so
// that the later dependent loads hit L2 instead of waiting on DRAM in turn.
BDDC_DEV void prefetch_l2(const double* p, int count) {
  const char* b = reinterpret_cast<const char*>(p);
  const long long bytes = (long long)count * 8;
  for (long long o = (long long)threadIdx.x * 128; o < bytes; o += (long long)blockDim.x * 128)
    asm volatile("prefetch.global.L2 [%0];\n" ::"l"(b + o));
}

// dst[i] = src[i], i < count (contiguous), four independent loads in flight per
// thread before the first store (generic-pointer stores would otherwise
// serialise the loads); no trailing barrier.
BDDC_DEV void copy_flat4(double* dst, const double* __restrict__ src, int count) {
  const int nt = blockDim.x;
  int i = threadIdx.x;
  for (; i + 3 * nt < count; i += 4 * nt) {
    const double a = src[i], b = src[i + nt], c = src[i + 2 * nt], d = src[i + 3 * nt];
    dst[i] = a;
    dst[i + nt] = b;
    dst[i + 2 * nt] = c;
    dst[i + 3 * nt] = d;
  }
  for (; i < count; i += nt) dst[i] = src[i];
}

// A <- (A + A^T)/2
BDDC_DEV void symmetrize(double* A, int ld, int n) {
  BLK_FOR_RC(n, n) {
    if (c > r) {
      double v = 0.5 * (A[r * ld + c] + A[c * ld + r]);
      A[r * ld + c] = v;
      A[c * ld + r] = v;
    }
  }
  __syncthreads();
}

template <bool TA, bool TB>
BDDC_DEV void gemm_t(double* C, int ldc, const double* A, int lda, const double* B, int ldb, int m,
                     int n, int k, double alpha, double beta) {
  BLK_FOR_RC(m, n) {
    double s = 0.0;
    for (int p = 0; p < k; ++p) {
      const double a = TA ? A[p * lda + r] : A[r * lda + p];
      const double b = TB ? B[c * ldb + p] : B[p * ldb + c];
      s = fma(a, b, s);
    }
    double v = alpha * s;
    if (beta != 0.0) v += beta * C[r * ldc + c];
    C[r * ldc + c] = v;
  }
  __syncthreads();
}

// Same contract on the DMMA pipe (mma.sync m8n8k4 f64): each warp computes up
// to kGT 16 x 8 output tiles at once (two 8x8 accumulators per tile sharing
// the B fragment), so 2 kGT independent DMMA chains hide the pipe latency;
// operands read straight from shared or global memory with zero-fill at the
// edges.
constexpr int kGT = 4;
template <bool TA, bool TB>
BDDC_DEV void gemm_mma_t(double* C, int ldc, const double* A, int lda, const double* B, int ldb,
                         int m, int n, int k, double alpha, double beta) {
  const int warp = (int)(threadIdx.x >> 5), lane = (int)(threadIdx.x & 31);
  const int nw = (int)(blockDim.x >> 5);
  const int g = lane >> 2, t = lane & 3;
  const int mt = (m + 15) >> 4, nt = (n + 7) >> 3;
  const int ntiles = mt * nt;
  for (int base = warp; base < ntiles; base += kGT * nw) {
    int ra[kGT], rb[kGT], cb[kGT];
    bool on[kGT];
    double x0[kGT], x1[kGT], y0[kGT], y1[kGT];
#pragma unroll
    for (int i = 0; i < kGT; ++i) {
      const int tile = base + i * nw;
      on[i] = tile < ntiles;
      const int tr = on[i] ? tile / nt : 0;
      const int r0 = tr * 16, c0 = on[i] ? (tile - tr * nt) * 8 : 0;
      ra[i] = r0 + g;
      rb[i] = r0 + 8 + g;
      cb[i] = c0 + g;
      x0[i] = x1[i] = y0[i] = y1[i] = 0.0;
    }
    for (int p = 0; p < k; p += 4) {
      const int kk = p + t;
      const bool kin = kk < k;
#pragma unroll
      for (int i = 0; i < kGT; ++i) {
        double a0 = 0.0, a1 = 0.0, bv = 0.0;
        if (on[i] && kin) {
          if (ra[i] < m) a0 = TA ? A[kk * lda + ra[i]] : A[ra[i] * lda + kk];
          if (rb[i] < m) a1 = TA ? A[kk * lda + rb[i]] : A[rb[i] * lda + kk];
          if (cb[i] < n) bv = TB ? B[cb[i] * ldb + kk] : B[kk * ldb + cb[i]];
        }
        dmma_8x8x4(x0[i], x1[i], a0, bv);
        dmma_8x8x4(y0[i], y1[i], a1, bv);
      }
    }
#pragma unroll
    for (int i = 0; i < kGT; ++i) {
      if (!on[i]) continue;
      const int cc = cb[i] - g + 2 * t;
      const double xs[2] = {x0[i], x1[i]}, ys[2] = {y0[i], y1[i]};
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (cc + h >= n) continue;
        if (ra[i] < m) {
          double v = alpha * xs[h];
          if (beta != 0.0) v += beta * C[ra[i] * ldc + cc + h];
          C[ra[i] * ldc + cc + h] = v;
        }
        if (rb[i] < m) {
          double v = alpha * ys[h];
          if (beta != 0.0) v += beta * C[rb[i] * ldc + cc + h];
          C[rb[i] * ldc + cc + h] = v;
        }
      }
    }
  }
  __syncthreads();
}

// C = beta*C + alpha*op(A)*op(B);  op(A) m x k, op(B) k x n.  C must not alias A/B.
BDDC_DEV void gemm(double* C, int ldc, const double* A, int lda, bool ta, const double* B, int ldb,
                   bool tb, int m, int n, int k, double alpha, double beta) {
  if (m >= 8 && n >= 8 && k >= 8) {
    if (!ta && !tb) gemm_mma_t<false, false>(C, ldc, A, lda, B, ldb, m, n, k, alpha, beta);
    else if (ta && !tb) gemm_mma_t<true, false>(C, ldc, A, lda, B, ldb, m, n, k, alpha, beta);
    else if (!ta && tb) gemm_mma_t<false, true>(C, ldc, A, lda, B, ldb, m, n, k, alpha, beta);
    else gemm_mma_t<true, true>(C, ldc, A, lda, B, ldb, m, n, k, alpha, beta);
    return;
  }
  if (!ta && !tb) gemm_t<false, false>(C, ldc, A, lda, B, ldb, m, n, k, alpha, beta);
  else if (ta && !tb) gemm_t<true, false>(C, ldc, A, lda, B, ldb, m, n, k, alpha, beta);
  else if (!ta && tb) gemm_t<false, true>(C, ldc, A, lda, B, ldb, m, n, k, alpha, beta);
  else gemm_t<true, true>(C, ldc, A, lda, B, ldb, m, n, k, alpha, beta);
}

// In-place scalar Gauss-Jordan inverse without pivoting.  Returns 0 on
// success, kNotPositiveDefinite if require_positive and a pivot <= 0 (the
// LDL^T pivots of a symmetric matrix: positive iff SPD, the cho_factor
// criterion), kSingularPivot on a zero / non-finite pivot.  rowbuf: 2n doubles.
BDDC_DEV int gj_inverse(double* A, int ld, int n, bool require_positive, double* rowbuf) {
  __shared__ int bad;
  if (tid() == 0) bad = 0;
  __syncthreads();
  for (int p = 0; p < n; ++p) {
    const double piv = A[p * ld + p];
    const bool fail = !(piv == piv) || piv == 0.0 || isinf(piv) || (require_positive && !(piv > 0.0));
    if (fail) {
      if (tid() == 0) bad = require_positive ? kNotPositiveDefinite : kSingularPivot;
      __syncthreads();
      break;
    }
    const double ip = 1.0 / piv;
    double* colbuf = rowbuf + n;
    for (int c = tid(); c < n; c += nth()) {
      rowbuf[c] = (c == p) ? ip : A[p * ld + c] * ip;
      colbuf[c] = A[c * ld + p];
    }
    __syncthreads();
    BLK_FOR_RC(n, n) {
      if (r == p) {
        A[r * ld + c] = rowbuf[c];
      } else {
        const double f = colbuf[r];
        A[r * ld + c] = (c == p) ? -f * ip : A[r * ld + c] - f * rowbuf[c];
      }
    }
    __syncthreads();
  }
  int out = bad;
  __syncthreads();
  return out;
}

// Cholesky A = L L^T in place (lower triangle).  Returns false when a pivot
// is <= 0 or not finite (LAPACK potrf failure).
BDDC_DEV bool cholesky(double* A, int ld, int n) {
  // Right-looking with ONE barrier per column: step j updates the trailing
  // lower triangle with the unscaled column, A[r][c] -= A[r][j] A[c][j] / d_j
  // (column j is outside the trailing block, so nothing written in a step is
  // read in the same step); the columns are scaled by 1 / sqrt(d_j) at the end.
  // Every thread reads the same pivot after the barrier: uniform early exit.
  bool ok = true;
  for (int j = 0; j < n; ++j) {
    const double d = A[j * ld + j];
    if (!(d > 0.0) || isinf(d)) {
      ok = false;
      break;
    }
    const double id = 1.0 / d;
    const int m = n - j - 1;
    if (nth() == 256 && m <= 48) {
      // register-tiled (3 x 3 elements per thread of a 16 x 16 grid): the column
      // entries are read once per tile row / column instead of once per element
      const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
      double ar[3], ac[3];
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const int r = ty + 16 * q, c = tx + 16 * q;
        ar[q] = r < m ? A[(j + 1 + r) * ld + j] : 0.0;
        ac[q] = c < m ? A[(j + 1 + c) * ld + j] : 0.0;
      }
#pragma unroll
      for (int a3 = 0; a3 < 3; ++a3) {
        const int r = ty + 16 * a3;
        if (r >= m) continue;
#pragma unroll
        for (int bq = 0; bq < 3; ++bq) {
          const int c = tx + 16 * bq;
          if (c <= r) A[(j + 1 + r) * ld + j + 1 + c] -= ar[a3] * ac[bq] * id;
        }
      }
    } else {
      BLK_FOR_RC(m, m) {
        if (c <= r) {
          const int ri = j + 1 + r, ci = j + 1 + c;
          A[ri * ld + ci] -= A[ri * ld + j] * A[ci * ld + j] * id;
        }
      }
    }
    __syncthreads();
  }
  if (ok) {
    BLK_FOR_RC(n, n) {
      if (c <= r) {
        const double s = sqrt(A[c * ld + c]);
        if (c < r) A[r * ld + c] /= s;
      }
    }
    __syncthreads();
    for (int j = tid(); j < n; j += nth()) A[j * ld + j] = sqrt(A[j * ld + j]);
  }
  __syncthreads();
  return ok;
}

// Solve (L L^T) X = B in place for B (n x nrhs), L from cholesky().
BDDC_DEV void chol_solve(const double* L, int ld, int n, double* B, int ldb, int nrhs) {
  for (int j = 0; j < n; ++j) {  // forward
    const double d = L[j * ld + j];
    for (int c = tid(); c < nrhs; c += nth()) B[j * ldb + c] /= d;
    __syncthreads();
    const int m = n - j - 1;
    BLK_FOR_RC(m, nrhs) B[(j + 1 + r) * ldb + c] -= L[(j + 1 + r) * ld + j] * B[j * ldb + c];
    __syncthreads();
  }
  for (int j = n - 1; j >= 0; --j) {  // backward with L^T
    const double d = L[j * ld + j];
    for (int c = tid(); c < nrhs; c += nth()) B[j * ldb + c] /= d;
    __syncthreads();
    BLK_FOR_RC(j, nrhs) B[r * ldb + c] -= L[j * ld + r] * B[j * ldb + c];
    __syncthreads();
  }
}

// Forward substitution in place: B <- L^-1 B (L lower triangular, n x n; B n x nrhs).
BDDC_DEV void trsm_lower(const double* L, int ld, int n, double* B, int ldb, int nrhs) {
  for (int j = 0; j < n; ++j) {
    const double d = L[j * ld + j];
    for (int c = tid(); c < nrhs; c += nth()) B[j * ldb + c] /= d;
    __syncthreads();
    const int m = n - j - 1;
    BLK_FOR_RC(m, nrhs) B[(j + 1 + r) * ldb + c] -= L[(j + 1 + r) * ld + j] * B[j * ldb + c];
    __syncthreads();
  }
}

// Block-wide max reduction helper (returns the same value on all threads).
BDDC_DEV double block_max(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = tid() >> 5, l = tid() & 31, nw = (nth() + 31) >> 5;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double r = red[0];
  for (int i = 1; i < nw; ++i) r = fmax(r, red[i]);
  __syncthreads();
  return r;
}

BDDC_DEV double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = tid() >> 5, l = tid() & 31, nw = (nth() + 31) >> 5;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double r = 0.0;
  for (int i = 0; i < nw; ++i) r += red[i];
  __syncthreads();
  return r;
}

// Squared Frobenius norm of an m x n block (same value on all threads).
BDDC_DEV double frob2(const double* A, int ld, int m, int n, double* red) {
  double s = 0.0;
  BLK_FOR_RC(m, n) {
    double v = A[r * ld + c];
    s += v * v;
  }
  return block_sum(s, red);
}

// Symmetric eigendecomposition by cyclic parallel two-sided Jacobi
// (round-robin pairing).  A (n x n, symmetric) is destroyed; w gets the
// eigenvalues in ascending order; if V != nullptr its columns are the
// matching orthonormal eigenvectors.  cs: 2*(n+2) doubles of scratch,
// perm: 2*(n+2) ints of scratch (shared memory preferred).
// Each round is two barrier phases: rotation parameters for the n/2
// disjoint pairs, then one fused update in which every (pair_i, pair_j)
// 2x2 block of A gets J_i^T A J_j (rows and columns at once) and V gets V J.
// Returns false if the sweep limit was reached.
BDDC_DEV bool jacobi_eigh(double* A, int ld, int n, double* w, double* V, int ldv, double* cs,
                          int* perm, double* red) {
  if (V) set_identity(V, ldv, n, n);
  if (n <= 1) {
    if (n == 1 && tid() == 0) w[0] = A[0];
    __syncthreads();
    return true;
  }
  const int m = n + (n & 1);  // even player count; index n is a bye when n is odd
  const int half = m / 2;
  bool converged = false;
  for (int sweep = 0; sweep < 40; ++sweep) {
    // threshold Jacobi: rotate (p,q) only while |a_pq| exceeds both a relative
    // (1e-15 sqrt|a_pp a_qq|) and an absolute (1e-17 max|a_ii|) floor; a sweep
    // without rotations ends the iteration.
    double dmax = 0.0;
    for (int i = tid(); i < n; i += nth()) dmax = fmax(dmax, fabs(A[i * ld + i]));
    dmax = block_max(dmax, red);
    const double abs_floor = fmax(1e-17 * dmax, 1e-300);
    int sweep_rot = 0;
    for (int round = 0; round < m - 1; ++round) {
      // phase 1: rotation of each pair (p < q); q == n is the bye
      int rot = 0;
      for (int i = tid(); i < half; i += nth()) {
        int a = i - 1 + round;
        if (a >= m - 1) a -= m - 1;
        a = (i == 0) ? 0 : 1 + a;
        int b = m - 2 - i + round;
        if (b >= m - 1) b -= m - 1;
        b += 1;
        int p = min(a, b), q = max(a, b);
        double c = 1.0, s = 0.0;
        if (q < n) {
          const double apq = A[p * ld + q];
          const double app = A[p * ld + p], aqq = A[q * ld + q];
          if (fabs(apq) > abs_floor && fabs(apq) > 1e-15 * sqrt(fabs(app) * fabs(aqq))) {
            const double tau = (aqq - app) / (2.0 * apq);
            const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
            c = 1.0 / sqrt(1.0 + t * t);
            s = t * c;
            rot = 1;
          }
        }
        perm[2 * i] = p;
        perm[2 * i + 1] = q;
        cs[2 * i] = c;
        cs[2 * i + 1] = s;
      }
      if (!__syncthreads_or(rot)) continue;
      sweep_rot = 1;
      // phase 2: A_blk(i,j) <- J_i^T A_blk J_j for bi <= bj (mirrored to (j,i),
      // A stays exactly symmetric);  V(:, pair j) <- V(:, pair j) J_j
      for (int bi = (int)(threadIdx.x >> 5); bi < half; bi += (int)(blockDim.x >> 5)) {
        const int p = perm[2 * bi], q = perm[2 * bi + 1];
        const double ci = cs[2 * bi], si = cs[2 * bi + 1];
        const bool hq = q < n;
        for (int bj = bi + (int)(threadIdx.x & 31); bj < half; bj += 32) {
          const int pc = perm[2 * bj], qc = perm[2 * bj + 1];
          const double cj = cs[2 * bj], sj = cs[2 * bj + 1];
          if (si == 0.0 && sj == 0.0) continue;  // both identity: block unchanged
          const bool hqc = qc < n;
          const double a00 = A[p * ld + pc];
          const double a01 = hqc ? A[p * ld + qc] : 0.0;
          const double a10 = hq ? A[q * ld + pc] : 0.0;
          const double a11 = (hq && hqc) ? A[q * ld + qc] : 0.0;
          // rows: x0 = c a_p - s a_q ; x1 = s a_p + c a_q
          const double x00 = ci * a00 - si * a10, x01 = ci * a01 - si * a11;
          const double x10 = si * a00 + ci * a10, x11 = si * a01 + ci * a11;
          // cols: y[:,0] = c x[:,0] - s x[:,1] ; y[:,1] = s x[:,0] + c x[:,1]
          const double y00 = cj * x00 - sj * x01, y01 = sj * x00 + cj * x01;
          const double y10 = cj * x10 - sj * x11, y11 = sj * x10 + cj * x11;
          if (bi == bj) {
            A[p * ld + p] = y00;
            if (hq) {
              A[p * ld + q] = y01;
              A[q * ld + p] = y01;
              A[q * ld + q] = y11;
            }
          } else {
            A[p * ld + pc] = y00;
            A[pc * ld + p] = y00;
            if (hqc) {
              A[p * ld + qc] = y01;
              A[qc * ld + p] = y01;
            }
            if (hq) {
              A[q * ld + pc] = y10;
              A[pc * ld + q] = y10;
            }
            if (hq && hqc) {
              A[q * ld + qc] = y11;
              A[qc * ld + q] = y11;
            }
          }
        }
      }
      if (V) {
        for (int bj = (int)(threadIdx.x >> 5); bj < half; bj += (int)(blockDim.x >> 5)) {
          const int pc = perm[2 * bj], qc = perm[2 * bj + 1];
          if (qc >= n || cs[2 * bj + 1] == 0.0) continue;
          const double cj = cs[2 * bj], sj = cs[2 * bj + 1];
          for (int r = (int)(threadIdx.x & 31); r < n; r += 32) {
            const double vp = V[r * ldv + pc], vq = V[r * ldv + qc];
            V[r * ldv + pc] = cj * vp - sj * vq;
            V[r * ldv + qc] = sj * vp + cj * vq;
          }
        }
      }
      __syncthreads();
    }
    if (!sweep_rot) { converged = true; break; }
  }
  // ascending sort of the diagonal (rank by counting; ties by index)
  for (int i = tid(); i < n; i += nth()) {
    double di = A[i * ld + i];
    int rank = 0;
    for (int j = 0; j < n; ++j) {
      double dj = A[j * ld + j];
      rank += (dj < di) || (dj == di && j < i);
    }
    perm[i] = rank;
  }
  __syncthreads();
  for (int i = tid(); i < n; i += nth()) w[perm[i]] = A[i * ld + i];
  __syncthreads();
  if (V) {
    // permute columns of V in place through A as scratch
    BLK_FOR_RC(n, n) A[r * ld + perm[c]] = V[r * ldv + c];
    __syncthreads();
    copy(V, ldv, A, ld, n, n);
  }
  return converged;
}

// One-sided Jacobi (Hestenes): orthogonalise the q columns of X (p x q) in
// place by plane rotations; if Y != nullptr accumulate Y <- Y J (q x q,
// caller initialises).  Afterwards column norms are singular values.
BDDC_DEV bool onesided_jacobi(double* X, int ldx, int p, int q, double* Y, int ldy, double* cs,
                              int* perm, double* red) {
  if (q <= 1) return true;
  const int m = q + (q & 1), half = m / 2;
  bool converged = false;
  for (int sweep = 0; sweep < 60; ++sweep) {
    double maxcos = 0.0;
    for (int round = 0; round < m - 1; ++round) {
      for (int i = tid(); i < half; i += nth()) {
        int a = (i == 0) ? 0 : 1 + (i - 1 + round) % (m - 1);
        int b = 1 + (m - 2 - i + round) % (m - 1);
        perm[2 * i] = min(a, b);
        perm[2 * i + 1] = max(a, b);
      }
      __syncthreads();
      // column inner products, one warp per pair
      const int warp = tid() >> 5, lane = tid() & 31, nw = nth() >> 5;
      for (int i = warp; i < half; i += nw) {
        int u = perm[2 * i], v = perm[2 * i + 1];
        double al = 0.0, be = 0.0, ga = 0.0;
        if (v < q) {
          for (int r = lane; r < p; r += 32) {
            double xu = X[r * ldx + u], xv = X[r * ldx + v];
            al += xu * xu;
            be += xv * xv;
            ga += xu * xv;
          }
        }
        for (int o = 16; o > 0; o >>= 1) {
          al += __shfl_xor_sync(0xffffffffu, al, o);
          be += __shfl_xor_sync(0xffffffffu, be, o);
          ga += __shfl_xor_sync(0xffffffffu, ga, o);
        }
        if (lane == 0) {
          double c = 1.0, s = 0.0;
          if (v < q && ga != 0.0 && al > 0.0 && be > 0.0) {
            double rc = fabs(ga) / sqrt(al * be);
            maxcos = fmax(maxcos, rc);
            if (rc > 1e-15) {
              double zeta = (be - al) / (2.0 * ga);
              double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
              c = 1.0 / sqrt(1.0 + t * t);
              s = c * t;
            }
          }
          cs[2 * i] = c;
          cs[2 * i + 1] = s;
        }
      }
      __syncthreads();
      for (int idx = tid(); idx < half * p; idx += nth()) {
        int i = idx / p, r = idx - i * p;
        int u = perm[2 * i], v = perm[2 * i + 1];
        double c = cs[2 * i], s = cs[2 * i + 1];
        if (v >= q || s == 0.0) continue;
        double xu = X[r * ldx + u], xv = X[r * ldx + v];
        X[r * ldx + u] = c * xu - s * xv;
        X[r * ldx + v] = s * xu + c * xv;
      }
      if (Y) {
        for (int idx = tid(); idx < half * q; idx += nth()) {
          int i = idx / q, r = idx - i * q;
          int u = perm[2 * i], v = perm[2 * i + 1];
          double c = cs[2 * i], s = cs[2 * i + 1];
          if (v >= q || s == 0.0) continue;
          double yu = Y[r * ldy + u], yv = Y[r * ldy + v];
          Y[r * ldy + u] = c * yu - s * yv;
          Y[r * ldy + v] = s * yu + c * yv;
        }
      }
      __syncthreads();
    }
    // warp-level maxima were written only by lane 0 threads; reduce them
    double mc = block_max(maxcos, red);
    if (mc <= 1e-15) { converged = true; break; }
  }
  return converged;
}

// Q (n x n) orthogonal whose first r rows are the given orthonormal rows
// U (r x n, ldu) and whose remaining rows complete an orthonormal basis,
// built from Householder reflectors of U^T.  H: n x n scratch,
// vbuf: n doubles scratch.
BDDC_DEV void complete_basis(const double* U, int ldu, int r, int n, double* Q, int ldq, double* H,
                             int ldh, double* vbuf, double* red) {
  // H <- U^T (n x r) in its first r columns, then QR by Householder
  for (int idx = tid(); idx < n * r; idx += nth()) {
    int i = idx / r, j = idx - i * r;
    H[i * ldh + j] = U[j * ldu + i];
  }
  // Qacc (stored in Q as an n x n matrix, columns = basis) starts as I
  set_identity(Q, ldq, n, n);
  __syncthreads();
  for (int j = 0; j < r; ++j) {
    // v = x - alpha e_j on rows j..n-1 of column j
    double ss = 0.0;
    for (int i = j + tid(); i < n; i += nth()) ss += H[i * ldh + j] * H[i * ldh + j];
    ss = block_sum(ss, red);
    const double x0 = H[j * ldh + j];
    const double alpha = (x0 >= 0.0 ? -1.0 : 1.0) * sqrt(ss);
    for (int i = tid(); i < n; i += nth())
      vbuf[i] = (i < j) ? 0.0 : (i == j ? x0 - alpha : H[i * ldh + j]);
    __syncthreads();
    double vn = 0.0;
    for (int i = j + tid(); i < n; i += nth()) vn += vbuf[i] * vbuf[i];
    vn = block_sum(vn, red);
    if (vn > 0.0) {
      const double beta = 2.0 / vn;
      // apply to remaining columns of H (j..r-1): H <- (I - beta v v^T) H
      for (int c = j + tid(); c < r; c += nth()) {
        double d = 0.0;
        for (int i = j; i < n; ++i) d += vbuf[i] * H[i * ldh + c];
        d *= beta;
        for (int i = j; i < n; ++i) H[i * ldh + c] -= d * vbuf[i];
      }
      // accumulate Qacc <- Qacc (I - beta v v^T): rows of Qacc
      for (int rr = tid(); rr < n; rr += nth()) {
        double d = 0.0;
        for (int i = j; i < n; ++i) d += Q[rr * ldq + i] * vbuf[i];
        d *= beta;
        for (int i = j; i < n; ++i) Q[rr * ldq + i] -= d * vbuf[i];
      }
    }
    __syncthreads();
  }
  // Qacc columns r.. complete span(U^T); write Q rows: [U; Qacc[:, r:]^T]
  for (int idx = tid(); idx < n * n; idx += nth()) {
    int i = idx / n, c = idx - i * n;
    H[i * ldh + c] = Q[i * ldq + c];
  }
  __syncthreads();
  for (int idx = tid(); idx < n * n; idx += nth()) {
    int rr = idx / n, c = idx - rr * n;
    Q[rr * ldq + c] = (rr < r) ? U[rr * ldu + c] : H[c * ldh + rr];
  }
  __syncthreads();
}


// ---------------------------------------------------------------------------
// Symmetric tridiagonal route: Householder reduction, bisection for all
// eigenvalues, inverse iteration for a chosen subset of eigenvectors, and
// back-transformation.  Used by the certified pencil fast path, which needs
// every eigenvalue but only the eigenvectors of the selected (lambda >= theta)
// modes.
// ---------------------------------------------------------------------------

// In place: A (n x n symmetric, lower triangle used) -> T = Q^T A Q with
// d (n), e (n-1); Householder vectors v_k (v_k[0] = 1 implicit) stored in
// A[k+2:n, k], scalars in tau[k].  work: 2n doubles.
BDDC_DEV void tridiagonalize(double* A, int ld, int n, double* d, double* e, double* tau,
                             double* work, double* red) {
  // Three barriers per Householder step: the column norm and p.v are reduced
  // redundantly inside every warp (shuffles) instead of with block reductions.
  (void)red;
  double* v = work;       // n
  double* p = work + n;   // n
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int k = 0; k < n - 2; ++k) {
    const int m = n - k - 1;  // length of the column below the diagonal
    double ss = 0.0;
    for (int i = lane; i < m - 1; i += 32) {
      const double x = A[(k + 2 + i) * ld + k];
      ss += x * x;
    }
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    const double alpha = A[(k + 1) * ld + k];
    double t, beta;
    if (ss == 0.0) {
      t = 0.0;
      beta = alpha;
    } else {
      beta = -copysign(sqrt(alpha * alpha + ss), alpha);
      t = (beta - alpha) / beta;
    }
    const double scal = (ss == 0.0) ? 0.0 : 1.0 / (alpha - beta);
    for (int i = tid(); i < m; i += nth())
      v[i] = (i == 0) ? 1.0 : A[(k + 1 + i) * ld + k] * scal;
    if (tid() == 0) {
      tau[k] = t;
      e[k] = beta;
    }
    // (no barrier here: the product below reads v straight from column k of A,
    // which this step only overwrites after the next barrier)
    if (t != 0.0) {
      if (nth() == 256 && m <= 48) {
        // Register-tiled form for the common size (shared-memory bandwidth is what
        // bounds this loop): thread (ty, tx) of a 16 x 16 grid owns the 3 x 3
        // elements (ty + 16 a, tx + 16 b); v and p are read once per row / column
        // of the tile instead of once per element (the update does the same
        // operations per element as the general form below).
        const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
        const double* vcol = A + (k + 1) * ld + k;
        double vc[3], s3[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int bq = 0; bq < 3; ++bq) {
          const int c = tx + 16 * bq;
          vc[bq] = c < m ? (c == 0 ? 1.0 : vcol[c * ld] * scal) : 0.0;
        }
#pragma unroll
        for (int a3 = 0; a3 < 3; ++a3) {
          const int r = ty + 16 * a3;
          if (r < m) {
            const double* ar = A + (k + 1 + r) * ld + k + 1;
#pragma unroll
            for (int bq = 0; bq < 3; ++bq) {
              const int c = tx + 16 * bq;
              if (c < m) s3[a3] += ar[c] * vc[bq];
            }
          }
        }
        // sum over the 16 threads of a row group (same ty: one half-warp)
#pragma unroll
        for (int a3 = 0; a3 < 3; ++a3) {
#pragma unroll
          for (int o = 8; o > 0; o >>= 1) s3[a3] += __shfl_xor_sync(0xffffffffu, s3[a3], o);
          const int r = ty + 16 * a3;
          if (tx == 0 && r < m) p[r] = t * s3[a3];
        }
        __syncthreads();
        double pv = 0.0;
        for (int i = lane; i < m; i += 32) pv += p[i] * v[i];
        for (int o = 16; o > 0; o >>= 1) pv += __shfl_xor_sync(0xffffffffu, pv, o);
        const double hc = 0.5 * t * pv;
        double vr[3], wr[3], wc[3];
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          const int r = ty + 16 * q, c = tx + 16 * q;
          vr[q] = r < m ? v[r] : 0.0;
          wr[q] = r < m ? p[r] - hc * vr[q] : 0.0;
          wc[q] = c < m ? p[c] - hc * vc[q] : 0.0;
        }
#pragma unroll
        for (int a3 = 0; a3 < 3; ++a3) {
          const int r = ty + 16 * a3;
          if (r >= m) continue;
          double* ar = A + (k + 1 + r) * ld + k + 1;
#pragma unroll
          for (int bq = 0; bq < 3; ++bq) {
            const int c = tx + 16 * bq;
            if (c < m) ar[c] -= vr[a3] * wc[bq] + wr[a3] * vc[bq];
          }
        }
      } else {
      // p = t * A22 v   (A22 = A[k+1:, k+1:], symmetric: use full stored block);
      // 4 lanes per row, each a strided quarter of the columns (short
      // dependency chains instead of one warp-wide reduction per row)
      for (int q0 = 0; q0 < 4 * m; q0 += nth()) {  // uniform trip count: full-warp shuffles
        const int q = q0 + tid(), r = q >> 2, part = q & 3;
        double s = 0.0;
        if (q < 4 * m) {
          const double* ar = A + (k + 1 + r) * ld + k + 1;
          const double* vc = A + (k + 1) * ld + k;
          for (int c = part; c < m; c += 4) s += ar[c] * (c == 0 ? 1.0 : vc[c * ld] * scal);
        }
        s += __shfl_xor_sync(0xffffffffu, s, 1);
        s += __shfl_xor_sync(0xffffffffu, s, 2);
        if (q < 4 * m && part == 0) p[r] = t * s;
      }
      __syncthreads();
      double pv = 0.0;
      for (int i = lane; i < m; i += 32) pv += p[i] * v[i];
      for (int o = 16; o > 0; o >>= 1) pv += __shfl_xor_sync(0xffffffffu, pv, o);
      const double hc = 0.5 * t * pv;
      // w = p - hc v ; A22 -= v w^T + w v^T
      BLK_FOR_RC(m, m) {
        const double wr = p[r] - hc * v[r], wc = p[c] - hc * v[c];
        A[(k + 1 + r) * ld + k + 1 + c] -= v[r] * wc + wr * v[c];
      }
      }
    }
    // keep v_k below the subdiagonal for the back-transformation (column k is
    // outside A22: no conflict with the update); each thread stores the entries
    // it computed itself
    for (int i = 1 + tid(); i < m; i += nth()) A[(k + 1 + i) * ld + k] *= scal;
    __syncthreads();
  }
  for (int i = tid(); i < n; i += nth()) d[i] = A[i * ld + i];
  if (tid() == 0 && n >= 2) e[n - 2] = A[(n - 1) * ld + n - 2];
  if (tid() == 0 && n >= 2) tau[n - 2] = 0.0;
  __syncthreads();
}

// Sturm count: number of eigenvalues of T strictly below x.
// q_i = d_i - x - e_(i-1)^2 / q_(i-1) with |q| >= pivmin (normal numbers):
// the reciprocal is the MUFU approximation plus two Newton steps (a few ulps,
// i.e. a relative perturbation of e^2 of that size -- the recurrence stays
// backward stable; only the signs are used).
BDDC_DEV double fast_rcp(double q) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
  r = fma(r, fma(-q, r, 1.0), r);
  r = fma(r, fma(-q, r, 1.0), r);
  return r;
}

BDDC_DEV int sturm_count(const double* d, const double* e, int n, double x, double pivmin) {
  int cnt = 0;
  double q = d[0] - x;
  if (fabs(q) < pivmin) q = -pivmin;
  if (q < 0.0) ++cnt;
  for (int i = 1; i < n; ++i) {
    q = d[i] - x - e[i - 1] * e[i - 1] * fast_rcp(q);
    if (fabs(q) < pivmin) q = -pivmin;
    if (q < 0.0) ++cnt;
  }
  return cnt;
}

// All eigenvalues of T in ascending order (w), one thread per eigenvalue,
// bisection to machine precision.
BDDC_DEV void tridiag_eigvals(const double* d, const double* e, int n, double* w, double* red) {
  double lo = 0.0, hi = 0.0, emax = 0.0;
  for (int i = tid(); i < n; i += nth()) {
    const double r = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i < n - 1 ? fabs(e[i]) : 0.0);
    lo = fmin(lo, d[i] - r);
    hi = fmax(hi, d[i] + r);
    if (i < n - 1) emax = fmax(emax, e[i] * e[i]);
  }
  lo = -block_max(-lo, red);
  hi = block_max(hi, red);
  emax = block_max(emax, red);
  const double nrm = fmax(fabs(lo), fabs(hi));
  const double pivmin = fmax(1e-300, 1e-300 * emax);
  lo -= 2.2e-16 * nrm * n + 1e-300;
  hi += 2.2e-16 * nrm * n + 1e-300;
  const double atol = 1e-17 * nrm + 1e-300;
  // multisection: a group of G lanes per eigenvalue evaluates G Sturm counts
  // per step (G+1 subintervals, log2(G+1) bits per step instead of 1)
  int G = 1;
  while (G < 8 && n * (2 * G) <= nth()) G *= 2;
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31, gl = lane & (G - 1), gbase = lane & ~(G - 1);
  const int ngroups = nth() / G;
  for (int j = tid() / G;; j += ngroups) {
    const bool active = j < n;
    if (!__any_sync(full, active)) break;
    double a = lo, b = hi;
    bool done = !active;
    for (int it = 0; it < 200; ++it) {
      if (!done && b - a <= 2.2e-16 * fmax(fabs(a), fabs(b)) + atol) done = true;
      if (__all_sync(full, done)) break;
      const double h = (b - a) / (double)(G + 1);
      const int cnt = done ? 0 : sturm_count(d, e, n, a + h * (double)(gl + 1), pivmin);
      int q = G;  // first subinterval end with more than j eigenvalues below
      for (int l = 0; l < G; ++l) {
        const int cl = __shfl_sync(full, cnt, gbase + l);
        if (q == G && cl > j) q = l;
      }
      if (!done) {
        const double na = (q == 0) ? a : a + h * (double)q;
        const double nb = (q == G) ? b : a + h * (double)(q + 1);
        if (!(na > a) && !(nb < b)) done = true;
        a = na;
        b = nb;
      }
    }
    if (active && gl == 0) w[j] = 0.5 * (a + b);
  }
  __syncthreads();
}

// (T - lam I) = P L U by Gaussian elimination with partial pivoting on the
// tridiagonal (single thread; u0,u1,u2,ml: n doubles each, pv: n ints).  Zero
// pivots are replaced by +-tiny; u0 returns the RECIPROCAL pivots, so that the
// repeated solves of an inverse iteration need no division.
BDDC_DEV void tridiag_shift_factor(const double* d, const double* e, int n, double lam, double tiny,
                                   double* u0, double* u1, double* u2, double* ml, int* pv) {
  for (int i = 0; i < n; ++i) {
    u0[i] = d[i] - lam;
    u1[i] = (i < n - 1) ? e[i] : 0.0;
    u2[i] = 0.0;
  }
  for (int k = 0; k < n - 1; ++k) {
    const double sub = e[k];
    if (fabs(sub) > fabs(u0[k])) {
      const double a = u0[k], b = u1[k], c = u2[k];
      const double dn = u0[k + 1], s1 = u1[k + 1];
      const double isub = 1.0 / sub;
      const double l = a * isub;
      u0[k] = isub;
      u1[k] = dn;
      u2[k] = s1;
      u0[k + 1] = b - l * dn;
      u1[k + 1] = c - l * s1;
      ml[k] = l;
      pv[k] = 1;
    } else {
      if (u0[k] == 0.0) u0[k] = tiny;
      const double ip = 1.0 / u0[k];
      const double l = sub * ip;
      u0[k] = ip;
      u0[k + 1] -= l * u1[k];
      u1[k + 1] -= l * u2[k];
      ml[k] = l;
      pv[k] = 0;
    }
  }
  if (u0[n - 1] == 0.0) u0[n - 1] = tiny;
  u0[n - 1] = 1.0 / u0[n - 1];
}

// x <- (T - lam I)^-1 x with the factors of tridiag_shift_factor
BDDC_DEV void tridiag_shift_solve(int n, double* x, const double* u0, const double* u1,
                                  const double* u2, const double* ml, const int* pv) {
  for (int k = 0; k < n - 1; ++k) {
    if (pv[k]) {
      const double t = x[k];
      x[k] = x[k + 1];
      x[k + 1] = t - ml[k] * x[k + 1];
    } else {
      x[k + 1] -= ml[k] * x[k];
    }
  }
  for (int i = n - 1; i >= 0; --i) {
    double s = x[i];
    if (i + 1 < n) s -= u1[i] * x[i + 1];
    if (i + 2 < n) s -= u2[i] * x[i + 2];
    x[i] = s * u0[i];
  }
}

// Eigenvectors of T for the eigenvalues w[idx[0..k-1]], one of kIILanes
// threads per cluster of close eigenvalues (|gap| <= 1e-3 ||T||), inverse
// iteration with Gram-Schmidt inside a cluster (LAPACK dstein strategy).
// X: n x k, columns = unit eigenvectors of T.  scratch: 5 n doubles per lane,
// iscratch: n ints per lane.
constexpr int kIILanes = 4;
BDDC_DEV void tridiag_eigvecs(const double* d, const double* e, int n, const double* w,
                              const int* idx, int k, double* X, double* scratch, int* iscratch) {
  if (threadIdx.x < kIILanes) {
    double tn = 0.0;
    for (int i = 0; i < n; ++i)
      tn = fmax(tn, fabs(d[i]) + (i > 0 ? fabs(e[i - 1]) : 0.0) + (i < n - 1 ? fabs(e[i]) : 0.0));
    const double tiny = fmax(2.2e-16 * tn, 1e-300);
    // cluster starts: lane handles clusters in order
    int cl = 0;
    for (int j = 0; j < k; ++j) {
      const bool start = (j == 0) || fabs(w[idx[j]] - w[idx[j - 1]]) > 1e-3 * tn;
      if (start) ++cl;
      if ((cl - 1) % kIILanes != (int)threadIdx.x) continue;
      int j0 = j;  // first member of this cluster
      while (j0 > 0 && !(fabs(w[idx[j0]] - w[idx[j0 - 1]]) > 1e-3 * tn)) --j0;
      double* x = scratch + threadIdx.x * 5 * n;
      double* u0 = x + n;
      double* u1 = u0 + n;
      double* u2 = u1 + n;
      double* ml = u2 + n;
      int* pv = iscratch + threadIdx.x * n;
      const double lam = w[idx[j]] + (j - j0) * 10.0 * tiny;  // separate equal shifts
      for (int i = 0; i < n; ++i) x[i] = 1.0 + 0.37 * sin(1.0 + 0.7 * i + 1.3 * (j - j0));
      // an isolated eigenvalue (gap > 1e-3 ||T|| to both spectral neighbours,
      // bisection-accurate shift)
      // converges to machine precision in two solves; clusters get five
      const int wi = idx[j];
      const bool isolated = (j == j0) && (wi == 0 || w[wi] - w[wi - 1] > 1e-3 * tn) &&
                            (wi == n - 1 || w[wi + 1] - w[wi] > 1e-3 * tn);
      const int iters = isolated ? 3 : 5;
      tridiag_shift_factor(d, e, n, lam, tiny, u0, u1, u2, ml, pv);  // once per shift
      for (int it = 0; it < iters; ++it) {
        tridiag_shift_solve(n, x, u0, u1, u2, ml, pv);
        // orthogonalise against the earlier members of the cluster
        for (int q = j0; q < j; ++q) {
          double dot = 0.0;
          for (int i = 0; i < n; ++i) dot += X[i * k + q] * x[i];
          for (int i = 0; i < n; ++i) x[i] -= dot * X[i * k + q];
        }
        double nrm = 0.0;
        for (int i = 0; i < n; ++i) nrm += x[i] * x[i];
        nrm = sqrt(nrm);
        const double inv = nrm > 0.0 ? 1.0 / nrm : 0.0;
        for (int i = 0; i < n; ++i) x[i] *= inv;
      }
      for (int i = 0; i < n; ++i) X[i * k + j] = x[i];
    }
  }
  __syncthreads();
}

// Y <- Q Y for the Householder Q of tridiagonalize() (Y: n x k, ld ldy).
BDDC_DEV void apply_householder(const double* A, int ld, int n, const double* tau, double* Y,
                                int ldy, int k) {
  for (int j = (int)(threadIdx.x >> 5); j < k; j += (int)(blockDim.x >> 5)) {
    const int lane = threadIdx.x & 31;
    for (int s = n - 3; s >= 0; --s) {
      const double t = tau[s];
      if (t == 0.0) continue;
      // v = [1; A[s+2:, s]] acting on rows s+1..n-1
      double dot = 0.0;
      for (int i = lane; i < n - s - 1; i += 32)
        dot += (i == 0 ? 1.0 : A[(s + 1 + i) * ld + s]) * Y[(s + 1 + i) * ldy + j];
      for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
      dot *= t;
      for (int i = lane; i < n - s - 1; i += 32)
        Y[(s + 1 + i) * ldy + j] -= dot * (i == 0 ? 1.0 : A[(s + 1 + i) * ld + s]);
      __syncwarp();
    }
  }
  __syncthreads();
}

}  // namespace blk
}  // namespace bddc
