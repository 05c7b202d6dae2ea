// Register-resident block Gauss-Jordan inverse of one <= 64 x 64 matrix per
// 256-thread CTA (the pivot-block inverse of the blocked eliminations and the
// per-slot glob Schur blocks).
#pragma once
#include "common.cuh"
#include "tile_mma.cuh"

#ifndef GJ_PROF
#define GJ_PROF_INIT
#define GJ_PROF(i)
#endif

namespace bddc {

// barrier of the 256 threads running reg_gj64: a named barrier, so that the
// first 256 threads of a larger CTA can run the inverse on their own
BDDC_DEV void gj_sync256() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

// reciprocal on the dependent pivot chain: hardware approximation plus two
// Newton steps (a few ulps; zero / non-finite pivots are flagged separately)
BDDC_DEV double gj_rcp(double q) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
  r = fma(r, fma(-q, r, 1.0), r);
  r = fma(r, fma(-q, r, 1.0), r);
  return r;
}

struct RegGjSmem {
  double rowb[2][4][kTile];
  double colb[2][4][kTile];
  int bad;
};

struct MmaGjSmem {
  double R[2][4][kTile];     // pivot rows (double-buffered by step parity)
  double F[2][kTile][4];     // pivot columns
  double U[4][68];           // Mi * R (pivot columns: I + Mi); stride 68: conflict-free B fragments
  double pv[kTile];          // scalar pivots (written to piv at the end)
  int bad;
};

// Inverse of the w x w (w <= 64) matrix M (leading dimension L) by
// Gauss-Jordan without pivoting, written to out (leading dimension ldo).
// Needs blockDim.x == 256.  Returns true (in every thread) when a pivot is
// zero / non-finite, or <= 0 with require_positive (the LDL^T pivots: the
// cho_factor criterion).  piv: the w scalar pivots (may be null).
BDDC_DEV bool reg_gj64_fma(const double* __restrict__ M, long long L, int w,
                           double* __restrict__ out, long long ldo, int require_positive,
                           double* __restrict__ piv, RegGjSmem& sm) {
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


// Same inverse with the rank-4 updates on the DMMA pipe.  The matrix lives in
// DMMA accumulator fragments: warp w owns rows 8w..8w+7, thread (g, t) holds
// (8w + g, 8j + 2t + h) for j < 8, h < 2.  Called by exactly 256 threads
// (threadIdx.x < 256; all barriers are the named barrier gj_sync256).
// Step s (pivots p = 4s..4s+3):
//   publish pivot rows R (owner warp) and pivot columns F (all warps);
//   Mi = R[:, p:p+4]^-1 (one thread: the 4x4 Gauss-Jordan, scalar pivots);
//   U = Mi R with U[:, p:p+4] = I + Mi, so that the single update
//   M -= F U (one m8n8k4 DMMA per 8x8 tile) also produces the new pivot
//   columns -F Mi; the pivot rows are then overwritten with U (Mi on the
//   pivot block).
BDDC_DEV bool reg_gj64(const double* __restrict__ M, long long L, int w, double* __restrict__ out,
                       long long ldo, int require_positive, double* __restrict__ piv,
                       MmaGjSmem& sm, int max_steps = 1 << 30) {
  GJ_PROF_INIT
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int row = 8 * warp + g;
  double c[8][2];
#pragma unroll
  for (int j = 0; j < 8; ++j)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int col = 8 * j + 2 * t + h;
      c[j][h] = (row < w && col < w) ? M[(long long)row * L + col] : (row == col ? 1.0 : 0.0);
    }
  bool bad_any = false;
  const int nsteps = min((w + 3) >> 2, max_steps);
  GJ_PROF(36);
  for (int s = 0; s < nsteps; ++s) {
    const int par = s & 1, p = 4 * s, pw = s >> 1, g0 = 4 * (s & 1);
    // publish pivot rows (owner warp) and pivot columns (tile jp = pw, lanes holding them)
    if (warp == pw && g >= g0 && g < g0 + 4) {
#pragma unroll
      for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) sm.R[par][g - g0][8 * j + 2 * t + h] = c[j][h];
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (j != pw) continue;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int cc = 2 * t + h - g0;
        if (cc >= 0 && cc < 4) sm.F[par][row][cc] = c[j][h];
      }
    }
    gj_sync256();
    GJ_PROF(32);
    // 4x4 Gauss-Jordan of the pivot block in every warp (lane 4i+j holds Mi[i][j],
    // lanes 16..31 mirror lanes 0..15): no shared-memory round trip for Mi
    double m;
    {
      // (the pivot bookkeeping stays out of this dependent chain: every lane
      // holds the same pivot, so the validity test is uniform and branch-free;
      // the pivots go to shared memory once per step and to piv at the end)
      const int i = (lane >> 2) & 3, jj = lane & 3;
      m = sm.R[par][i][p + jj];
      double pvq[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double pv = __shfl_sync(0xffffffffu, m, 5 * q);
        const double rq = __shfl_sync(0xffffffffu, m, 4 * q + jj);
        const double cq = __shfl_sync(0xffffffffu, m, 4 * i + q);
        pvq[q] = pv;
        bad_any |= (p + q < w) &&
                   (!(pv == pv) || pv == 0.0 || isinf(pv) || (require_positive && !(pv > 0.0)));
        const double ip = gj_rcp(pv);
        if (i == q) m = (jj == q) ? ip : rq * ip;
        else m = (jj == q) ? -cq * ip : m - cq * rq * ip;
      }
      if (threadIdx.x < 4) {
        double v = pvq[0];
#pragma unroll
        for (int q = 1; q < 4; ++q)
          if ((int)threadIdx.x == q) v = pvq[q];
        sm.pv[p + threadIdx.x] = v;
      }
    }
    GJ_PROF(33);
    {  // U = Mi R, pivot columns I + Mi: one value per thread (i is warp-uniform)
      const int i = threadIdx.x >> 6, col = threadIdx.x & 63;
      const double m0 = __shfl_sync(0xffffffffu, m, 4 * i), m1 = __shfl_sync(0xffffffffu, m, 4 * i + 1);
      const double m2 = __shfl_sync(0xffffffffu, m, 4 * i + 2), m3 = __shfl_sync(0xffffffffu, m, 4 * i + 3);
      double u;
      if (col >= p && col < p + 4) {
        const int k = col - p;
        u = (k == 0 ? m0 : k == 1 ? m1 : k == 2 ? m2 : m3) + (i == k ? 1.0 : 0.0);
      } else {
        u = m0 * sm.R[par][0][col] + m1 * sm.R[par][1][col] + m2 * sm.R[par][2][col] +
            m3 * sm.R[par][3][col];
      }
      sm.U[i][col] = u;
    }
    // the pivot-block values a pivot-row lane needs: Mi[g - g0][2t + h - (p - 8 pw)]
    double mp[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int gi = (g - g0) & 3, k = (2 * t + h - g0) & 3;
      mp[h] = __shfl_sync(0xffffffffu, m, 4 * gi + k);
    }
    gj_sync256();
    GJ_PROF(34);
    // M -= F U on the tensor pipe
    const double a = -sm.F[par][row][t];
#pragma unroll
    for (int j = 0; j < 8; ++j) dmma_8x8x4(c[j][0], c[j][1], a, sm.U[t][8 * j + g]);
    // pivot rows <- U (Mi on the pivot block)
    if (warp == pw && g >= g0 && g < g0 + 4) {
#pragma unroll
      for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int col = 8 * j + 2 * t + h;
          c[j][h] = (col >= p && col < p + 4) ? mp[h] : sm.U[g - g0][col];
        }
    }
    GJ_PROF(35);
  }
  gj_sync256();
#pragma unroll
  for (int j = 0; j < 8; ++j)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int col = 8 * j + 2 * t + h;
      if (row < w && col < w) out[(long long)row * ldo + col] = c[j][h];
    }
  if (piv)
    for (int i = threadIdx.x; i < min(w, 4 * nsteps); i += 256) piv[i] = sm.pv[i];
  gj_sync256();  // sm reusable after return
  GJ_PROF(37);
  return bad_any;  // the same value in every thread
}

}  // namespace bddc
