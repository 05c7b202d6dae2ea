// 64x64 fp64 tile GEMM on the DMMA pipe (mma.sync m8n8k4.f64, sm_100a).
//
// One CTA of 128 threads (2x2 warps, 32x32 per warp = 4x4 DMMA tiles)
// computes   C[m x n] = beta*C + alpha * A[m x K] * B[K x n]   with
// m, n <= 64 and K <= 64.  A and B are staged whole into shared memory
// (row stride 68 doubles: conflict-free DMMA fragment loads), so B may alias
// C when one CTA owns every row of that C tile (in-place W = P*W updates).
#pragma once
#include "common.cuh"

namespace bddc {

constexpr int kTile = 64;
constexpr int kTileStride = 68;
constexpr int kTileThreads = 128;

struct TileSmem {
  double A[kTile][kTileStride];
  double B[kTile][kTileStride];
};

// Cooperative fill of a 64 x K4 tile from a row-major source, zero padded.
BDDC_DEV void tile_load(double (*dst)[kTileStride], const double* src, long long ld, int rows,
                        int cols, int rows_pad, int cols_pad) {
  for (int idx = threadIdx.x; idx < rows_pad * cols_pad; idx += kTileThreads) {
    int r = idx / cols_pad, c = idx - r * cols_pad;
    dst[r][c] = (r < rows && c < cols) ? src[(long long)r * ld + c] : 0.0;
  }
}

BDDC_DEV void tile_mma(double* C, long long ldc, int m, int n, const double* A, long long lda,
                       const double* B, long long ldb, int K, double alpha, double beta,
                       TileSmem& sm) {
  const int K4 = (K + 3) & ~3;
  tile_load(sm.A, A, lda, m, K, kTile, K4);
  tile_load(sm.B, B, ldb, K, n, K4, kTile);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int k0 = 0; k0 < K4; k0 += 4) {
    double a[4], b[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = sm.A[wm + i * 8 + g][k0 + t];
#pragma unroll
    for (int j = 0; j < 4; ++j) b[j] = sm.B[k0 + t][wn + j * 8 + g];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = wm + i * 8 + g;
    if (r >= m) continue;
    double* crow = C + (long long)r * ldc;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = wn + j * 8 + 2 * t;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (c + h < n) {
          double v = alpha * acc[i][j][h];
          if (beta != 0.0) v += beta * crow[c + h];
          crow[c + h] = v;
        }
      }
    }
  }
}

}  // namespace bddc
