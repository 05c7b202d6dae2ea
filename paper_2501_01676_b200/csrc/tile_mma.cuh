// BM x 64 fp64 tile GEMM on the DMMA pipe (mma.sync m8n8k4.f64, sm_100a).
//
// One CTA ((BM/32) x (64/kWN) warps, 32 x kWN per warp; default kWN = 16,
// 8 warps, <= 64 registers so 4 CTAs fit per SM — measured best with
// tools/bench_tile.py) computes   C[m x n] = beta*C + alpha * A[m x K] * B[K x n]   with
// m <= BM, n <= 64 and K <= 64.  A and B stream through shared memory in
// K-chunks of 16 with a 3-stage cp.async pipeline (16-byte copies when the
// source is 16-byte aligned, 8-byte otherwise; out-of-range elements
// zero-filled); C is prefetched into L2 at the start and read once, in the
// epilogue (out = alpha * acc + beta * C), so the first DMMAs wait only on the
// first K-chunk.  B may alias C when one CTA
// owns every row of that C tile and beta == 0 (in-place W = P*W updates):
// all of B is read before the epilogue writes.
#pragma once
#include "common.cuh"

namespace bddc {

#ifndef BDDC_KC
#define BDDC_KC 16
#endif
#ifndef BDDC_KSTAGES
#define BDDC_KSTAGES 3
#endif
#ifndef BDDC_TILE_MINB
#define BDDC_TILE_MINB 4   // <= 64 registers: 4 CTAs x 8 warps per SM (tools/bench_tile.py)
#endif

#ifndef BDDC_C_LATE
#define BDDC_C_LATE 1      // zero-start accumulators, C prefetched to L2 and added in the epilogue
                           // (0: accumulators start from (beta/alpha) C; measured ~2 % slower)
#endif

#ifndef BDDC_WN
#define BDDC_WN 16         // 32x16 warp tiles, 8 warps per 64x64 CTA tile
#endif

constexpr int kTile = 64;
constexpr int kWN = BDDC_WN;                       // warp tile width (32 or 16)
constexpr int kNJ = kWN / 8;                        // DMMA tiles per warp along n
constexpr int kTileThreads = 2 * 32 * (64 / kWN);  // BM = 64: 2 x (64 / kWN) warps
constexpr int kKC = BDDC_KC;          // K chunk
constexpr int kStages = BDDC_KSTAGES;
constexpr int kTileMinBlocks = BDDC_TILE_MINB;
constexpr int kAS = kKC + 4;     // A smem row stride (doubles): conflict-free fragments
constexpr int kBS = kTile + 4;   // B smem row stride

// BM x 64 output tile: (BM/32) x (64/kWN) warps, each warp 32 x kWN
// (4 x kWN/8 DMMA m8n8k4 tiles).
template <int BM>
struct TileSmemT {
  double A[kStages][BM][kAS];
  double B[kStages][kKC][kBS];
};
using TileSmem = TileSmemT<64>;

BDDC_DEV void cp_async8(double* dst, const double* src, bool valid) {
  unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(src),
               "r"(valid ? 8 : 0));
}

BDDC_DEV void cp_async16(double* dst, const double* src, int valid_doubles) {
  unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(src),
               "r"(valid_doubles * 8));
}

BDDC_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }

template <int N>
BDDC_DEV void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// async load of K-chunk `kc` of A (BM x kKC) and B (kKC x 64) into stage `st`
template <int BM>
BDDC_DEV void tile_issue_chunk(TileSmemT<BM>& sm, int st, int kc, const double* A, long long lda,
                               const double* B, long long ldb, int m, int n, int K, bool a16,
                               bool b16) {
  constexpr int NT = (BM / 32) * (64 / kWN) * 32;
  const int k0 = kc * kKC;
  if (a16) {
    for (int idx = threadIdx.x; idx < BM * (kKC / 2); idx += NT) {
      const int r = idx / (kKC / 2), c = (idx - r * (kKC / 2)) * 2;
      const int kk = k0 + c;
      int valid = (r < m) ? max(0, min(2, K - kk)) : 0;
      const double* src = valid ? A + (long long)r * lda + kk : A;
      cp_async16(&sm.A[st][r][c], src, valid);
    }
  } else {
    for (int idx = threadIdx.x; idx < BM * kKC; idx += NT) {
      const int r = idx / kKC, c = idx - r * kKC;
      const bool valid = r < m && k0 + c < K;
      cp_async8(&sm.A[st][r][c], valid ? A + (long long)r * lda + k0 + c : A, valid);
    }
  }
  if (b16) {
    for (int idx = threadIdx.x; idx < kKC * (kTile / 2); idx += NT) {
      const int r = idx / (kTile / 2), c = (idx - r * (kTile / 2)) * 2;
      int valid = (k0 + r < K) ? max(0, min(2, n - c)) : 0;
      const double* src = valid ? B + (long long)(k0 + r) * ldb + c : B;
      cp_async16(&sm.B[st][r][c], src, valid);
    }
  } else {
    for (int idx = threadIdx.x; idx < kKC * kTile; idx += NT) {
      const int r = idx / kTile, c = idx - r * kTile;
      const bool valid = k0 + r < K && c < n;
      cp_async8(&sm.B[st][r][c], valid ? B + (long long)(k0 + r) * ldb + c : B, valid);
    }
  }
}

// Thin edge tile (n <= 8 columns or m <= 8 rows, e.g. the two extra dofs of
// nB = 386 = 6 * 64 + 2): every warp owns one 8 x 8 DMMA accumulator (row
// block `warp` for thin columns, column block `warp` for thin rows) and reads
// its fragments straight from global memory, so the tile costs 1/8 of a full
// one.  Same contract as tile_mma_t (B may alias C: all reads precede the
// writes).  Not inlined: the hot path's register allocation stays untouched.
template <int BM>
__device__ __noinline__ void tile_mma_thin(double* C, long long ldc, int m, int n, const double* A,
                                           long long lda, const double* B, long long ldb, int K,
                                           double alpha, double beta, double* Ct, long long ldct,
                                           double tsign) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const bool thin_cols = n <= 8;
  const int r0 = thin_cols ? 8 * warp : 0, c0 = thin_cols ? 0 : 8 * warp;
  const int ra = r0 + g, cb = c0 + g;
  const bool on = r0 < m && c0 < n;  // warp-uniform
  double x0 = 0.0, x1 = 0.0;
  if (on) {
#pragma unroll 4
    for (int p = 0; p < K; p += 4) {
      const int kk = p + t;
      const double a = (kk < K && ra < m) ? A[(long long)ra * lda + kk] : 0.0;
      const double b = (kk < K && cb < n) ? B[(long long)kk * ldb + cb] : 0.0;
      dmma_8x8x4(x0, x1, a, b);
    }
  }
  const int cc = c0 + 2 * t;
  double v[2] = {alpha * x0, alpha * x1};
  if (on && ra < m && beta != 0.0) {
#pragma unroll
    for (int h = 0; h < 2; ++h)
      if (cc + h < n) v[h] = fma(beta, C[(long long)ra * ldc + cc + h], v[h]);
  }
  __syncthreads();  // every read of B (which may alias C) is done
  if (on && ra < m) {
#pragma unroll
    for (int h = 0; h < 2; ++h)
      if (cc + h < n) {
        C[(long long)ra * ldc + cc + h] = v[h];
        if (Ct != nullptr) Ct[(long long)(cc + h) * ldct + ra] = tsign * v[h];
      }
  }
}

template <int BM>
BDDC_DEV void tile_mma_t(double* C, long long ldc, int m, int n, const double* A, long long lda,
                         const double* B, long long ldb, int K, double alpha, double beta,
                         TileSmemT<BM>& sm, double* Ct = nullptr, long long ldct = 0,
                         double tsign = 1.0) {
  constexpr int WNW = 64 / kWN;  // warps along n
  if (n <= 8 || m <= 8) {  // CTA-uniform
    tile_mma_thin<BM>(C, ldc, m, n, A, lda, B, ldb, K, alpha, beta, Ct, ldct, tsign);
    return;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp / WNW) * 32, wn = (warp % WNW) * kWN;  // (BM/32) x WNW warps
  const int nchunks = (K + kKC - 1) / kKC;
  const bool a16 = ((reinterpret_cast<uintptr_t>(A) | (uintptr_t)(lda * 8)) & 15) == 0;
  const bool b16 = ((reinterpret_cast<uintptr_t>(B) | (uintptr_t)(ldb * 8)) & 15) == 0;
#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) {
    if (s < nchunks) tile_issue_chunk(sm, s, s, A, lda, B, ldb, m, n, K, a16, b16);
    cp_async_commit();
  }
  double acc[4][kNJ][2];
  const bool c16 = ((reinterpret_cast<uintptr_t>(C) | (uintptr_t)(ldc * 8)) & 15) == 0;
#if BDDC_C_LATE
  // accumulators start at zero so the first DMMAs wait only on the first
  // chunk; C is prefetched into L2 now and read in the epilogue
  if (beta != 0.0) {
    constexpr int NT = (BM / 32) * (64 / kWN) * 32;
    for (int idx = threadIdx.x; idx < BM * 4; idx += NT) {
      const int r = idx >> 2, c = (idx & 3) * 16;
      if (r < m && c < n)
        asm volatile("prefetch.global.L2 [%0];\n" ::"l"(C + (long long)r * ldc + c));
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < kNJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#else
  // accumulators start from (beta/alpha) C: C is read once, early, while the
  // first chunks are in flight
  const double cscale = (beta != 0.0) ? beta / alpha : 0.0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = wm + i * 8 + g;
#pragma unroll
    for (int j = 0; j < kNJ; ++j) {
      const int c = wn + j * 8 + 2 * t;
      if (cscale != 0.0 && r < m && c + 1 < n && c16) {
        const double2 v = *reinterpret_cast<const double2*>(C + (long long)r * ldc + c);
        acc[i][j][0] = cscale * v.x;
        acc[i][j][1] = cscale * v.y;
      } else {
#pragma unroll
        for (int h = 0; h < 2; ++h)
          acc[i][j][h] = (cscale != 0.0 && r < m && c + h < n) ? cscale * C[(long long)r * ldc + c + h] : 0.0;
      }
    }
  }
#endif
  for (int kc = 0; kc < nchunks; ++kc) {
    cp_async_wait<kStages - 2>();
    __syncthreads();
    const int nxt = kc + kStages - 1;
    if (nxt < nchunks) tile_issue_chunk(sm, nxt % kStages, nxt, A, lda, B, ldb, m, n, K, a16, b16);
    cp_async_commit();
    const int st = kc % kStages;
    const int kmax = min(kKC, K - kc * kKC);
    if (kmax == kKC) {
      // full chunk: unrolled, so the fragment loads of step k0 + 4 are issued
      // while the DMMAs of step k0 run
#pragma unroll
      for (int k0 = 0; k0 < kKC; k0 += 4) {
        double a[4], b[kNJ];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = sm.A[st][wm + i * 8 + g][k0 + t];
#pragma unroll
        for (int j = 0; j < kNJ; ++j) b[j] = sm.B[st][k0 + t][wn + j * 8 + g];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < kNJ; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
      }
    } else {
      for (int k0 = 0; k0 < kmax; k0 += 4) {
        double a[4], b[kNJ];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = sm.A[st][wm + i * 8 + g][k0 + t];
#pragma unroll
        for (int j = 0; j < kNJ; ++j) b[j] = sm.B[st][k0 + t][wn + j * 8 + g];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < kNJ; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
      }
    }
  }
  cp_async_wait<0>();
  __syncthreads();  // every read of B (which may alias C) is done
  // final values alpha * acc (+ beta * C when C is read late)
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = wm + i * 8 + g;
#pragma unroll
    for (int j = 0; j < kNJ; ++j) {
      const int c = wn + j * 8 + 2 * t;
#if BDDC_C_LATE
      if (beta != 0.0 && r < m) {
        if (c + 1 < n && c16) {
          const double2 v = *reinterpret_cast<const double2*>(C + (long long)r * ldc + c);
          acc[i][j][0] = fma(alpha, acc[i][j][0], beta * v.x);
          acc[i][j][1] = fma(alpha, acc[i][j][1], beta * v.y);
        } else {
#pragma unroll
          for (int h = 0; h < 2; ++h)
            acc[i][j][h] = (c + h < n) ? fma(alpha, acc[i][j][h], beta * C[(long long)r * ldc + c + h])
                                       : alpha * acc[i][j][h];
        }
        continue;
      }
#endif
      acc[i][j][0] *= alpha;
      acc[i][j][1] *= alpha;
    }
  }
  if (Ct != nullptr) {
    // mirrored copy: Ct[c][r] = tsign * C[r][c], staged through shared memory
    // (the pipeline buffers are free now) so both stores are coalesced
    static_assert(sizeof(TileSmemT<BM>) >= sizeof(double) * 64 * 65, "staging tile");
    double* st = reinterpret_cast<double*>(&sm);
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < kNJ; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = wm + i * 8 + g, c = wn + j * 8 + 2 * t + h;
          st[c * 65 + r] = tsign * acc[i][j][h];
        }
    __syncthreads();
    constexpr int NT = (BM / 32) * (64 / kWN) * 32;
    for (int idx = threadIdx.x; idx < 64 * BM; idx += NT) {
      const int c = idx / BM, r = idx - c * BM;
      if (c < n && r < m) Ct[(long long)c * ldct + r] = st[c * 65 + r];
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = wm + i * 8 + g;
    if (r >= m) continue;
    double* crow = C + (long long)r * ldc;
#pragma unroll
    for (int j = 0; j < kNJ; ++j) {
      const int c = wn + j * 8 + 2 * t;
      if (c + 1 < n && c16) {
        *reinterpret_cast<double2*>(crow + c) = make_double2(acc[i][j][0], acc[i][j][1]);
      } else {
#pragma unroll
        for (int h = 0; h < 2; ++h)
          if (c + h < n) crow[c + h] = acc[i][j][h];
      }
    }
  }
}

BDDC_DEV void tile_mma(double* C, long long ldc, int m, int n, const double* A, long long lda,
                       const double* B, long long ldb, int K, double alpha, double beta,
                       TileSmem& sm, double* Ct = nullptr, long long ldct = 0,
                       double tsign = 1.0) {
  tile_mma_t<64>(C, ldc, m, n, A, lda, B, ldb, K, alpha, beta, sm, Ct, ldct, tsign);
}

}  // namespace bddc
