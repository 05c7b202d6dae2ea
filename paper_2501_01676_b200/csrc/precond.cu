// BDDC preconditioner setup and apply, interface operator, coarse problem.
//
// Reference: solver.py:54-134 (setup), 138-209 (apply), 226-242 (S_hat, g_hat).
//
// Per subdomain i, in the glob-major local B order (each glob contiguous):
//   T_i  = blockdiag_g(Q_g D_g^(i)T)                    (transformed deluxe)
//   Sbar = Q_i S_i Q_i^T,  Z = (Sbar_dd)^-1 embedded (zero on primal rows/cols)
//   A_i  = T_i^T Z T_i                    local part of M^-1   (nB x nB)
//   G_i  = (E_P - E_P Sbar Z) T_i         coarse restriction   (n_p x nB)
//   N_i  = T_i^T (E_P - Z Sbar E_P)       coarse prolongation  (stored n_p x nB)
//   C_i  = Sbar_PP - Sbar_P: Z Sbar_:P    coarse contribution  (n_p x n_p)
// so that M^-1 r = sum_i R_i^T (A_i R_i r + N_i u_P,i),
//         u_P = C^-1 sum_i P_i^T G_i R_i r     (C = sum_i P_i^T C_i P_i).
// This is algebraically the reference's Qhat^T Rtil^T Dtil Stil^-1 Dtil^T Rtil Qhat.
#include <cooperative_groups.h>

#include "common.cuh"
#include "bddc_b200.h"
#include "tile_mma.cuh"
#include "lu_solve.cuh"
#include "dense_block.cuh"

namespace cg = cooperative_groups;

namespace bddc {

struct SubGlobMap {
  const int* nB;
  const long long* soff;      // nB x nB matrices
  const long long* voff;      // nB vectors (prefix sum of nB)
  const int* pos2k;           // per local B position: index into sub_globs
  const int* sub_globs;       // glob id per (sub, k)
  const int* sub_glob_boff;   // block offset per (sub, k)
  const int* sub_glob_sh;     // sharer slot (into sh_* of the glob) per (sub, k)
  const int* gsize;           // per glob size
  const double* Q;            // per glob Q (n_g x n_g)
  const long long* q_off;
  const double* D;            // per (glob, sharer) D
  const long long* sh_doff;
};

// X = op(Qi) S op(Qi)^T style block transforms ------------------------------
// out[r][c] = sum_q L_blk(r)[r', q] * in[blk0(r) + q][c]      (left multiply)
//   mode 0: L = Q_g           mode 1: L = (Q_g D_g^T)^T = D_g Q_g^T
// Right multiplies are done as (left multiply on the transpose) by the caller
// through the `trans_in` / `trans_out` flags.
__device__ __forceinline__ double left_block_value(const SubGlobMap& m, int sub, int r, int q,
                                                   int mode) {
  const int k = m.pos2k[m.voff[sub] + r];
  const int g = m.sub_globs[k];
  const int bo = m.sub_glob_boff[k];
  const int ng = m.gsize[g];
  const int rr = r - bo;
  const double* Qg = m.Q + m.q_off[g];
  if (mode == 0) return Qg[rr * ng + q];
  // T^T[rr][q] = (Q D^T)^T[rr][q] = (D Q^T)[rr][q] = sum_a D[rr][a] Q[q][a]
  const double* Dg = m.D + m.sh_doff[m.sub_glob_sh[k]];
  double s = 0.0;
  for (int a = 0; a < ng; ++a) s += Dg[rr * ng + a] * Qg[q * ng + a];
  return s;
}

// out = L * in (in/out nB x nB, ld nB); if right: out = in * L^T.
// L is block diagonal with blocks given by left_block_value(mode).
__global__ void block_transform_kernel(SubGlobMap m, const double* __restrict__ in,
                                       double* __restrict__ out, int mode, int right) {
  const int b = blockIdx.y;
  const int n = m.nB[b];
  const double* X = in + m.soff[b];
  double* Y = out + m.soff[b];
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < (long long)n * n;
       idx += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(idx / n), c = (int)(idx - (long long)r * n);
    const int pivot = right ? c : r;
    const int k = m.pos2k[m.voff[b] + pivot];
    const int bo = m.sub_glob_boff[k];
    const int ng = m.gsize[m.sub_globs[k]];
    double s = 0.0;
    for (int q = 0; q < ng; ++q) {
      const double l = left_block_value(m, b, pivot, q, mode);
      s += right ? X[(long long)r * n + bo + q] * l : l * X[(long long)(bo + q) * n + c];
    }
    Y[idx] = s;
  }
}

// Block-diagonal transforms, one CTA per (glob block, subdomain):
//   left : out[blk, :] = L_blk * in[blk, :]
//   right: out[:, blk] = in[:, blk] * L_blk^T
// L_blk = Q_g (src 0) or TT_(g,s) = D_g^(s) Q_g^T (src 1).  in/out nB x nB.
constexpr int kBT_COLS = 32;
__global__ void __launch_bounds__(256) glob_block_kernel(SubGlobMap m,
                                                         const int* __restrict__ sub_glob_start,
                                                         const double* __restrict__ TT,
                                                         const double* __restrict__ in,
                                                         double* __restrict__ out, int src,
                                                         int right, int max_ng, int skip_ge) {
  extern __shared__ double smb[];
  const int b = blockIdx.y;
  const int k = sub_glob_start[b] + blockIdx.x;
  if (k >= sub_glob_start[b + 1]) return;
  const int n = m.nB[b];
  const int g = m.sub_globs[k];
  const int bo = m.sub_glob_boff[k];
  const int ng = m.gsize[g];
  if (ng >= skip_ge) return;  // large blocks go through glob_mma_kernel
  const double* L = src == 0 ? m.Q + m.q_off[g] : TT + m.sh_doff[m.sub_glob_sh[k]];
  const double* X = in + m.soff[b];
  double* Y = out + m.soff[b];
  const bool lsm = ng <= 64;
  double* Ls = smb;                       // ng x ng (when ng <= 64)
  double* Xt = smb + (lsm ? 64 * 64 : 0);  // tile: ng x kBT_COLS (left) or kBT_COLS x ng (right)
  if (lsm) {
    for (int i = threadIdx.x; i < ng * ng; i += blockDim.x) Ls[i] = L[i];
  }
  const double* Lp = lsm ? Ls : L;
  for (int t0 = 0; t0 < n; t0 += kBT_COLS) {
    const int tw = min(kBT_COLS, n - t0);
    __syncthreads();
    if (!right) {
      for (int i = threadIdx.x; i < ng * tw; i += blockDim.x) {
        const int q = i / tw, c = i - q * tw;
        Xt[q * kBT_COLS + c] = X[(long long)(bo + q) * n + t0 + c];
      }
    } else {
      for (int i = threadIdx.x; i < tw * ng; i += blockDim.x) {
        const int r = i / ng, q = i - r * ng;
        Xt[r * max_ng + q] = X[(long long)(t0 + r) * n + bo + q];
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < ng * tw; i += blockDim.x) {
      double s = 0.0;
      if (!right) {
        const int r = i / tw, c = i - r * tw;
        for (int q = 0; q < ng; ++q) s += Lp[r * ng + q] * Xt[q * kBT_COLS + c];
        Y[(long long)(bo + r) * n + t0 + c] = s;
      } else {
        const int r = i / ng, c = i - r * ng;
        for (int q = 0; q < ng; ++q) s += Xt[r * max_ng + q] * Lp[c * ng + q];
        Y[(long long)(t0 + r) * n + bo + c] = s;
      }
    }
  }
}

// DMMA version of the block-diagonal transforms: one CTA per (glob block of a
// subdomain, 64-wide tile of the free dimension, 64-chunk of the glob
// dimension), block products on the tensor pipe via tile_mma:
//   left : out[blk, tile] = L_blk * in[blk, tile]
//   right: out[tile, blk] = in[tile, blk] * L_blk^T   (B operand = L^T, from LT)
// L_blk = base + off[g] (by_slot = 0) or base + off[sub_glob_sh[k]] (by_slot = 1).
__global__ void __launch_bounds__(kTileThreads, kTileMinBlocks) glob_mma_kernel(
    const int* __restrict__ nB, const long long* __restrict__ soff,
    const int* __restrict__ sub_glob_start, int nsub, const int* __restrict__ sub_globs,
    const int* __restrict__ sub_glob_boff, const int* __restrict__ sub_glob_sh,
    const int* __restrict__ gsize, const double* __restrict__ L, const double* __restrict__ LT,
    const long long* __restrict__ loff, int by_slot, int right, const double* __restrict__ in,
    double* __restrict__ out, int tiles_per_item, int min_ng) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  TileSmem& sm = *reinterpret_cast<TileSmem*>(smem_raw);
  const int item = blockIdx.x / tiles_per_item, tile = blockIdx.x - item * tiles_per_item;
  const int rc = blockIdx.y;
  // subdomain owning glob item `item` (binary search in sub_glob_start)
  int lo = 0, hi = nsub;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (sub_glob_start[mid] <= item) lo = mid; else hi = mid;
  }
  const int b = lo;
  const int n = nB[b];
  const int g = sub_globs[item];
  const int ng = gsize[g];
  const int bo = sub_glob_boff[item];
  if (ng < min_ng || rc * 64 >= ng || tile * 64 >= n) return;
  const long long lo_off = loff[by_slot ? sub_glob_sh[item] : g];
  const double* X = in + soff[b];
  double* Y = out + soff[b];
  for (int kc = 0; kc < ng; kc += 64) {
    const int K = min(64, ng - kc);
    if (!right) {
      const int m = min(64, ng - rc * 64), nc = min(64, n - tile * 64);
      tile_mma(Y + (long long)(bo + rc * 64) * n + tile * 64, n, m, nc,
               L + lo_off + (long long)(rc * 64) * ng + kc, ng,
               X + (long long)(bo + kc) * n + tile * 64, n, K, 1.0, kc ? 1.0 : 0.0, sm);
    } else {
      const int m = min(64, n - tile * 64), nc = min(64, ng - rc * 64);
      tile_mma(Y + (long long)(tile * 64) * n + bo + rc * 64, n, m, nc,
               X + (long long)(tile * 64) * n + bo + kc, n,
               LT + lo_off + (long long)kc * ng + rc * 64, ng, K, 1.0, kc ? 1.0 : 0.0, sm);
    }
  }
}


// ---------------------------------------------------------------------------
// Change of basis in Householder form.  The preconditioner only needs a Q_g
// whose first r rows span the primal constraints of glob g (M^-1 is invariant
// under rotations inside the primal span and inside its complement), so Q_g
// is replaced by H_r ... H_1 from the Householder QR of Q_g[:r]^T.  Then
// Sbar = Q S Q^T costs 2 r n_g nB flops per glob block and side instead of a
// dense n_g x n_g block product.  Reflector j is stored as w_j = sqrt(beta_j) v_j
// (H_j = I - w_j w_j^T) in row j of the glob's n_g x n_g block of HV.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128) glob_reflectors_kernel(
    const int* __restrict__ kind, const int* __restrict__ gsize, const int* __restrict__ r,
    double* __restrict__ Q, const long long* __restrict__ q_off, double* __restrict__ HV,
    double* __restrict__ W, const long long* __restrict__ w_off) {
  extern __shared__ double rsm[];
  const int g = blockIdx.x;
  const int n = gsize[g];
  const int rr = kind[g] == 2 ? 0 : min(r[g], n);
  double* Qg = Q + q_off[g];
  double* Hg = HV + q_off[g];
  double* Wg = W + w_off[g];       // n x rr: Q_g[:rr]^T, reduced in place
  double* v = rsm;                 // n
  double* red = rsm + n;           // 4 warps
  if (rr == 0) return;             // Q_g = I (no constraint) or a vertex: untouched
  if (n == 1) {                    // [+-1] -> [1]: same span, no reflector
    if (threadIdx.x == 0) Qg[0] = 1.0;
    return;
  }
  for (int idx = threadIdx.x; idx < n * rr; idx += blockDim.x) {
    const int i = idx / rr, j = idx - i * rr;
    Wg[idx] = Qg[j * n + i];
  }
  __syncthreads();  // every read of Q_g before it is reset
  for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) Qg[idx] = (idx / n == idx % n) ? 1.0 : 0.0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int j = 0; j < rr; ++j) {
    double ss = 0.0;
    for (int i = j + threadIdx.x; i < n; i += blockDim.x) ss += Wg[i * rr + j] * Wg[i * rr + j];
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if (lane == 0) red[warp] = ss;
    __syncthreads();
    ss = red[0] + red[1] + red[2] + red[3];
    const double x0 = Wg[j * rr + j];
    const double alpha = (x0 >= 0.0 ? -1.0 : 1.0) * sqrt(ss);
    const double vn = ss - x0 * x0 + (x0 - alpha) * (x0 - alpha);
    const double beta = vn > 0.0 ? 2.0 / vn : 0.0;
    const double sb = sqrt(beta);
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const double vi = i < j ? 0.0 : (i == j ? x0 - alpha : Wg[i * rr + j]);
      v[i] = vi;
      Hg[j * n + i] = sb * vi;
    }
    __syncthreads();
    if (beta != 0.0) {
      for (int c = j + 1 + threadIdx.x; c < rr; c += blockDim.x) {  // W <- H_j W
        double d = 0.0;
        for (int i = j; i < n; ++i) d += v[i] * Wg[i * rr + c];
        d *= beta;
        for (int i = j; i < n; ++i) Wg[i * rr + c] -= d * v[i];
      }
      for (int row = threadIdx.x; row < n; row += blockDim.x) {  // Qacc <- Qacc H_j
        double d = 0.0;
        for (int i = j; i < n; ++i) d += Qg[row * n + i] * v[i];
        d *= beta;
        for (int i = j; i < n; ++i) Qg[row * n + i] -= d * v[i];
      }
    }
    __syncthreads();
  }
  // Q_g = Qacc^T = H_r ... H_1 (reflectors are symmetric)
  for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
    const int a = idx / n, b = idx - a * n;
    if (a < b) {
      const double t = Qg[a * n + b];
      Qg[a * n + b] = Qg[b * n + a];
      Qg[b * n + a] = t;
    }
  }
}

// Sbar = Q S Q^T with Q = blockdiag_g(H_r ... H_1), one CTA per subdomain:
// rows (left product, S -> Sbar) then columns (right product, in place).
__global__ void __launch_bounds__(256) transform_refl_kernel(
    const int* __restrict__ nB, const long long* __restrict__ soff,
    const int* __restrict__ sub_glob_start, const int* __restrict__ sub_globs,
    const int* __restrict__ sub_glob_boff, const int* __restrict__ kind,
    const int* __restrict__ gsize, const int* __restrict__ r, const double* __restrict__ HV,
    const long long* __restrict__ q_off, const double* __restrict__ S, double* __restrict__ Sbar) {
  const int b = blockIdx.x;
  const int n = nB[b];
  const double* Sb = S + soff[b];
  double* Tb = Sbar + soff[b];
  const int k0 = sub_glob_start[b], k1 = sub_glob_start[b + 1];
  // left: thread per column, every glob block of rows
  for (int c = threadIdx.x; c < n; c += blockDim.x) {
    for (int k = k0; k < k1; ++k) {
      const int g = sub_globs[k], ng = gsize[g], bo = sub_glob_boff[k];
      const int nref = (kind[g] == 2 || ng == 1) ? 0 : min(r[g], ng);
      if (nref == 0) {
        for (int i = 0; i < ng; ++i) Tb[(long long)(bo + i) * n + c] = Sb[(long long)(bo + i) * n + c];
        continue;
      }
      const double* Hg = HV + q_off[g];
      for (int j = 0; j < nref; ++j) {
        const double* src = j == 0 ? Sb : Tb;
        const double* w = Hg + j * ng;
        double d = 0.0;
        for (int i = j; i < ng; ++i) d += w[i] * src[(long long)(bo + i) * n + c];
        for (int i = 0; i < ng; ++i)
          Tb[(long long)(bo + i) * n + c] = src[(long long)(bo + i) * n + c] - (i < j ? 0.0 : d * w[i]);
      }
    }
  }
  __syncthreads();
  // right: warp per row, lanes along the glob's columns
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int row = warp; row < n; row += nw) {
    double* tr = Tb + (long long)row * n;
    for (int k = k0; k < k1; ++k) {
      const int g = sub_globs[k], ng = gsize[g], bo = sub_glob_boff[k];
      const int nref = (kind[g] == 2 || ng == 1) ? 0 : min(r[g], ng);
      const double* Hg = HV + q_off[g];
      for (int j = 0; j < nref; ++j) {
        const double* w = Hg + j * ng;
        double d = 0.0;
        for (int i = j + lane; i < ng; i += 32) d += tr[bo + i] * w[i];
        for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
        for (int i = j + lane; i < ng; i += 32) tr[bo + i] -= d * w[i];
        __syncwarp();
      }
    }
  }
}


// Sbar = Q S Q^T with Q in Householder form (reflectors HV, r per glob), the
// compact primal rows / columns of Sbar and the embedded dual block Z
// (identity on primal rows and columns) -- the inputs of the dual LU and the
// primal pieces:
//  left pass, one CTA per glob block that has reflectors: X = Q_g S[rows of g]
//  written into Z's rows (thread per column);
//  row pass, one warp per row of every subdomain: the row (from Z for rows of
//  reflected globs, else from S) is staged in shared memory, the right
//  reflectors of the subdomain's reflected globs only (refl_start / refl_k) are
//  applied, then the compact primal row / column entries and the embedded dual
//  block row are written.
__global__ void __launch_bounds__(256) transform_left_kernel(
    const int* __restrict__ nB, const long long* __restrict__ soff,
    const int* __restrict__ item_k, const int* __restrict__ item_sub,
    const int* __restrict__ sub_globs, const int* __restrict__ sub_glob_boff,
    const int* __restrict__ gsize, const int* __restrict__ r, const double* __restrict__ HV,
    const long long* __restrict__ q_off, const double* __restrict__ S, double* __restrict__ Z) {
  const int kk = item_k[blockIdx.x], b = item_sub[blockIdx.x];
  const int n = nB[b];
  const int g = sub_globs[kk], ng = gsize[g], bo = sub_glob_boff[kk];
  const double* Sb = S + soff[b] + (long long)bo * n;
  double* X = Z + soff[b] + (long long)bo * n;
  const int nref = min(r[g], ng);
  const double* Hg = HV + q_off[g];
  for (int c = threadIdx.x; c < n; c += blockDim.x) {
    for (int j = 0; j < nref; ++j) {
      const double* src = j == 0 ? Sb : X;
      const double* w = Hg + j * ng;
      double d = 0.0;
      for (int i = j; i < ng; ++i) d += w[i] * src[(long long)i * n + c];
      for (int i = 0; i < ng; ++i)
        X[(long long)i * n + c] = src[(long long)i * n + c] - (i < j ? 0.0 : d * w[i]);
    }
  }
}

__global__ void __launch_bounds__(256) transform_rows_kernel(
    const int* __restrict__ nB, const long long* __restrict__ soff,
    const long long* __restrict__ voff, const int* __restrict__ pos2k,
    const int* __restrict__ sub_globs, const int* __restrict__ sub_glob_boff,
    const int* __restrict__ kind, const int* __restrict__ gsize, const int* __restrict__ r,
    const double* __restrict__ HV, const long long* __restrict__ q_off,
    const int* __restrict__ refl_start, const int* __restrict__ refl_k,
    const int* __restrict__ pidx, const long long* __restrict__ poff,
    const double* __restrict__ S, double* __restrict__ Z, double* __restrict__ Srows,
    double* __restrict__ Scols, int max_nB) {
  extern __shared__ double rowsm[];
  const int b = blockIdx.y;
  const int n = nB[b];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int rho = blockIdx.x * nw + warp;
  if (rho >= n) return;
  double* xr = rowsm + (size_t)warp * max_nB;
  const int k = pos2k[voff[b] + rho];
  const int g = sub_globs[k];
  const bool left = !(kind[g] == 2 || gsize[g] == 1) && r[g] > 0;
  const double* src = (left ? Z : S) + soff[b] + (long long)rho * n;
  for (int c = lane; c < n; c += 32) xr[c] = src[c];
  __syncwarp();
  for (int q = refl_start[b]; q < refl_start[b + 1]; ++q) {
    const int k2 = refl_k[q];
    const int h = sub_globs[k2], nh = gsize[h], bh = sub_glob_boff[k2];
    const int nrh = min(r[h], nh);
    const double* Hh = HV + q_off[h];
    for (int j = 0; j < nrh; ++j) {
      const double* w = Hh + j * nh;
      double d = 0.0;
      for (int i = j + lane; i < nh; i += 32) d += xr[bh + i] * w[i];
      for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
      for (int i = j + lane; i < nh; i += 32) xr[bh + i] -= d * w[i];
      __syncwarp();
    }
  }
  const int* pi = pidx + voff[b];
  const int qr = pi[rho];
  double* Sr = Srows + poff[b];
  double* Sc = Scols + poff[b];
  double* zr = Z + soff[b] + (long long)rho * n;
  for (int c = lane; c < n; c += 32) {
    const double v = xr[c];
    const int qc = pi[c];
    if (qr >= 0) Sr[(long long)qr * n + c] = v;
    if (qc >= 0) Sc[(long long)qc * n + rho] = v;
    zr[c] = (qr >= 0 || qc >= 0) ? (rho == c ? 1.0 : 0.0) : v;
  }
}

// compact primal rows / columns of a full Sbar (dense-Q path)
__global__ void primal_extract_kernel(const int* __restrict__ nB, const long long* __restrict__ soff,
                                      const long long* __restrict__ voff,
                                      const int* __restrict__ pidx,
                                      const long long* __restrict__ poff,
                                      const double* __restrict__ Sbar, double* __restrict__ Srows,
                                      double* __restrict__ Scols) {
  const int b = blockIdx.y;
  const int n = nB[b];
  const int* pi = pidx + voff[b];
  const double* Sb = Sbar + soff[b];
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < (long long)n * n;
       idx += (long long)gridDim.x * blockDim.x) {
    const int rr = (int)(idx / n), c = (int)(idx - (long long)rr * n);
    const int qr = pi[rr], qc = pi[c];
    if (qr >= 0) Srows[poff[b] + (long long)qr * n + c] = Sb[idx];
    if (qc >= 0) Scols[poff[b] + (long long)qc * n + rr] = Sb[idx];
  }
}

// dst block = src block^T for square blocks (size[gidx[i]]) at off[i]
__global__ void transpose_blocks_kernel(const double* __restrict__ src, double* __restrict__ dst,
                                        const long long* __restrict__ off,
                                        const int* __restrict__ gidx,
                                        const int* __restrict__ gsize, int nblocks) {
  const int i = blockIdx.x;
  if (i >= nblocks) return;
  const int n = gsize[gidx ? gidx[i] : i];
  const double* s = src + off[i];
  double* d = dst + off[i];
  for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
    const int r = idx / n, c = idx - r * n;
    d[c * n + r] = s[idx];
  }
}

// Primal pieces, one CTA per subdomain, primal positions in chunks of kPC:
//   MP[p][r] = d(r,pc) - (Z Sbar)[r][pc]     (warp per row r of Z, coalesced)
//   RP[p][r] = d(r,pc) - (Sbar Z)[pc][r]     (thread per column r of Z, coalesced)
//   C_i[p][q] = Sbar[pr, :] . MP[q, :]
constexpr int kPC = 8;
__global__ void __launch_bounds__(256) primal_pieces2_kernel(
    const int* __restrict__ nB, const long long* __restrict__ soff, const int* __restrict__ pstart,
    const int* __restrict__ ppos, const long long* __restrict__ poff,
    const double* __restrict__ Sbar, const double* __restrict__ Z, double* __restrict__ MP,
    double* __restrict__ RP, double* __restrict__ Cl, const long long* __restrict__ coff,
    int max_nB) {
  extern __shared__ double smp[];
  const int b = blockIdx.x;
  const int n = nB[b];
  const int p0 = pstart[b], np = pstart[b + 1] - p0;
  if (np == 0) return;
  const double* S = Sbar + soff[b];
  const double* Zb = Z + soff[b];
  double* M = MP + poff[b];
  double* R = RP + poff[b];
  double* Sc = smp;                   // kPC x max_nB: Sbar[:, pc]
  double* Sr = smp + kPC * max_nB;    // kPC x max_nB: Sbar[pc, :]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int c0 = 0; c0 < np; c0 += kPC) {
    const int pc_n = min(kPC, np - c0);
    __syncthreads();
    for (int i = threadIdx.x; i < pc_n * n; i += blockDim.x) {
      const int p = i / n, k = i - p * n;
      const int pc = ppos[p0 + c0 + p];
      Sc[p * max_nB + k] = S[(long long)k * n + pc];
      Sr[p * max_nB + k] = S[(long long)pc * n + k];
    }
    __syncthreads();
    // MP: warp per row of Z
    for (int r = warp; r < n; r += nw) {
      double acc[kPC];
#pragma unroll
      for (int p = 0; p < kPC; ++p) acc[p] = 0.0;
      const double* zr = Zb + (long long)r * n;
      for (int k = lane; k < n; k += 32) {
        const double z = zr[k];
#pragma unroll
        for (int p = 0; p < kPC; ++p)
          if (p < pc_n) acc[p] += z * Sc[p * max_nB + k];
      }
#pragma unroll
      for (int p = 0; p < kPC; ++p) {
        double v = acc[p];
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0 && p < pc_n) {
          const int pc = ppos[p0 + c0 + p];
          M[(long long)(c0 + p) * n + r] = (r == pc ? 1.0 : 0.0) - v;
        }
      }
    }
    // RP: thread per column of Z
    for (int r = threadIdx.x; r < n; r += blockDim.x) {
      double acc[kPC];
#pragma unroll
      for (int p = 0; p < kPC; ++p) acc[p] = 0.0;
      for (int k = 0; k < n; ++k) {
        const double z = Zb[(long long)k * n + r];
#pragma unroll
        for (int p = 0; p < kPC; ++p)
          if (p < pc_n) acc[p] += Sr[p * max_nB + k] * z;
      }
#pragma unroll
      for (int p = 0; p < kPC; ++p)
        if (p < pc_n) {
          const int pc = ppos[p0 + c0 + p];
          R[(long long)(c0 + p) * n + r] = (r == pc ? 1.0 : 0.0) - acc[p];
        }
    }
  }
  __syncthreads();
  double* C = Cl + coff[b];
  for (int i = warp; i < np * np; i += nw) {
    const int p = i / np, q = i - p * np;
    const int pr = ppos[p0 + p];
    double v = 0.0;
    for (int k = lane; k < n; k += 32) v += S[(long long)pr * n + k] * M[(long long)q * n + k];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) C[i] = v;
  }
}

// precompute TT blocks: TTb[(g,s)] = D_g^(s) Q_g^T  (so T^T blocks), per sharer slot
__global__ void ttblock_kernel(const int* __restrict__ slot_glob, const int* __restrict__ gsize,
                               const double* __restrict__ Q, const long long* __restrict__ q_off,
                               const double* __restrict__ D, const long long* __restrict__ sh_doff,
                               double* __restrict__ TT, int n_slots) {
  const int s = blockIdx.x;
  if (s >= n_slots) return;
  const int g = slot_glob[s];
  const int n = gsize[g];
  // TT = D Q^T on the DMMA pipe (dense_block.cuh)
  blk::gemm(TT + sh_doff[s], n, D + sh_doff[s], n, false, Q + q_off[g], n, true, n, n, n, 1.0, 0.0);
}

// Dense transformed deluxe weights per subdomain in the reference's nodal B
// order (solver.py:86-90): Dbar_b[pos, pos] = Q_g D_g^(b) Q_g^T for every glob
// slot (g, b), pos = nodal local positions of g's nodes in b (nodal[] maps a
// glob-major local position to the nodal one).  W: slot-layout scratch.
// Dbar must be zeroed by the caller (entries outside glob blocks stay 0).
__global__ void dbar_kernel(const int* __restrict__ slot_glob, const int* __restrict__ slot_sub,
                            const int* __restrict__ gsize, const int* __restrict__ sh_boff,
                            const long long* __restrict__ sh_doff, const double* __restrict__ Q,
                            const long long* __restrict__ q_off, const double* __restrict__ TT,
                            const int* __restrict__ nB, const long long* __restrict__ soff,
                            const long long* __restrict__ voff, const int* __restrict__ nodal,
                            double* __restrict__ W, double* __restrict__ Dbar) {
  const int s = blockIdx.x;
  const int g = slot_glob[s], b = slot_sub[s];
  const int n = gsize[g];
  double* Ws = W + sh_doff[s];
  blk::gemm(Ws, n, Q + q_off[g], n, false, TT + sh_doff[s], n, false, n, n, n, 1.0, 0.0);
  __syncthreads();
  const int nb = nB[b];
  const int* pos = nodal + voff[b] + sh_boff[s];
  double* Db = Dbar + soff[b];
  for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
    const int r = idx / n, c = idx - r * n;
    Db[(long long)pos[r] * nb + pos[c]] = Ws[idx];
  }
}

// out_b = X_b^T for square batched matrices (ld = n)
__global__ void transpose_batched_kernel(const double* __restrict__ X,
                                         const long long* __restrict__ soff,
                                         const int* __restrict__ nn, double* __restrict__ out) {
  const int b = blockIdx.y;
  const int n = nn[b];
  const double* A = X + soff[b];
  double* T = out + soff[b];
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < (long long)n * n;
       idx += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(idx / n), c = (int)(idx - (long long)r * n);
    T[(long long)c * n + r] = A[idx];
  }
}

// out = TT_blockdiag * in  (left) or in * TT_blockdiag^T (right), TT from ttblock_kernel
__global__ void tt_transform_kernel(SubGlobMap m, const double* __restrict__ TT,
                                    const double* __restrict__ in, double* __restrict__ out,
                                    int right, int transpose_block) {
  const int b = blockIdx.y;
  const int n = m.nB[b];
  const double* X = in + m.soff[b];
  double* Y = out + m.soff[b];
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < (long long)n * n;
       idx += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(idx / n), c = (int)(idx - (long long)r * n);
    const int pivot = right ? c : r;
    const int k = m.pos2k[m.voff[b] + pivot];
    const int bo = m.sub_glob_boff[k];
    const int ng = m.gsize[m.sub_globs[k]];
    const double* Tb = TT + m.sh_doff[m.sub_glob_sh[k]];
    const int pr = pivot - bo;
    double s = 0.0;
    for (int q = 0; q < ng; ++q) {
      const double l = transpose_block ? Tb[q * ng + pr] : Tb[pr * ng + q];
      s += right ? X[(long long)r * n + bo + q] * l : l * X[(long long)(bo + q) * n + c];
    }
    Y[idx] = s;
  }
}

// Zin <- Sbar with primal rows/cols replaced by identity; Csym <- sym(Zin)
__global__ void dual_embed_kernel(const int* __restrict__ nB, const long long* __restrict__ soff,
                                  const long long* __restrict__ voff,
                                  const unsigned char* __restrict__ primal_mask,
                                  const double* __restrict__ Sbar, double* __restrict__ Zin,
                                  double* __restrict__ Csym) {
  const int b = blockIdx.y;
  const int n = nB[b];
  const unsigned char* pm = primal_mask + voff[b];
  const double* S = Sbar + soff[b];
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < (long long)n * n;
       idx += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(idx / n), c = (int)(idx - (long long)r * n);
    double v, vs;
    if (pm[r] || pm[c]) {
      v = vs = (r == c) ? 1.0 : 0.0;
    } else {
      v = S[idx];
      vs = 0.5 * (v + S[(long long)c * n + r]);
    }
    Zin[soff[b] + idx] = v;
    if (Csym) Csym[soff[b] + idx] = vs;
  }
}



// ---------------------------------------------------------------------------
// dual solves with the blocked LU of the embedded dual block (lu_solve.cuh)
// ---------------------------------------------------------------------------
// P_k^-1 (kept per panel by schur_eliminate) into the diagonal blocks
__global__ void lu_diag_pinv_kernel(double* __restrict__ LU, const long long* __restrict__ soff,
                                    const int* __restrict__ nB, const double* __restrict__ pinv,
                                    long long pinv_stride, long long step_stride) {
  const int b = blockIdx.y, k = blockIdx.x;
  const int n = nB[b], k0 = k * 64;
  if (k0 >= n) return;
  const int w = min(64, n - k0);
  const double* P = pinv + (long long)k * step_stride + (long long)b * pinv_stride;
  double* D = LU + soff[b] + (long long)k0 * n + k0;
  for (int idx = threadIdx.x; idx < w * w; idx += blockDim.x) {
    const int r = idx / w, c = idx - r * w;
    D[(long long)r * n + c] = P[r * 64 + c];
  }
}

// coarse restriction alone, cvals = G x with x = u[perm] (one CTA per subdomain, warp
// per primal row): lets the coarse solve start while the local solves still run
__global__ void __launch_bounds__(256) primal_restrict_kernel(
    const int* __restrict__ nB, const long long* __restrict__ voff,
    const int* __restrict__ iface_perm, const double* __restrict__ u,
    const int* __restrict__ pstart, const long long* __restrict__ poff,
    const double* __restrict__ G, double* __restrict__ cvals) {
  extern __shared__ double rsm[];
  const int b = blockIdx.x;
  const int n = nB[b];
  const int np = pstart[b + 1] - pstart[b];
  if (np == 0) return;
  const long long v0 = voff[b];
  for (int j = threadIdx.x; j < n; j += blockDim.x) rsm[j] = u[iface_perm[v0 + j]];
  __syncthreads();
  lus::rows_gemv<1>(G + poff[b], n, np, n, rsm, cvals + pstart[b], 1.0, 0.0);
}

// local part of M^-1 and the coarse restriction, one CTA per subdomain:
//   x = r[perm];  cvals = G x;  t = TT^T x (primal entries zeroed);  t = Sdd^-1 t (LU);
//   y = TT t        (= A_i x with A_i = TT Z TT^T, without forming A_i)
__global__ void __launch_bounds__(256) local_solve_kernel(
    const int* __restrict__ nB, const long long* __restrict__ soff,
    const long long* __restrict__ voff, const int* __restrict__ iface_perm,
    const double* __restrict__ LU, const int* __restrict__ pos2k,
    const int* __restrict__ sub_globs, const int* __restrict__ sub_glob_boff,
    const int* __restrict__ sub_glob_sh, const int* __restrict__ gsize,
    const long long* __restrict__ sh_doff, const double* __restrict__ TT,
    const unsigned char* __restrict__ primal_mask, const double* __restrict__ u,
    double* __restrict__ y, const int* __restrict__ pstart, const long long* __restrict__ poff,
    const double* __restrict__ G, double* __restrict__ cvals) {
  extern __shared__ double lsm[];
  const int b = blockIdx.x;
  const int n = nB[b];
  double* xs = lsm;             // n
  double* ts = lsm + n;         // n
  double* tmp = lsm + 2 * n;    // 64
  const long long v0 = voff[b];
  for (int j = threadIdx.x; j < n; j += blockDim.x) xs[j] = u[iface_perm[v0 + j]];
  __syncthreads();
  const int np = pstart[b + 1] - pstart[b];
  if (np && G) lus::rows_gemv<1>(G + poff[b], n, np, n, xs, cvals + pstart[b], 1.0, 0.0);
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double s = 0.0;
    if (!primal_mask[v0 + i]) {
      const int k = pos2k[v0 + i];
      const int bo = sub_glob_boff[k], ng = gsize[sub_globs[k]];
      const double* Tb = TT + sh_doff[sub_glob_sh[k]];
      const int ii = i - bo;
      for (int j = 0; j < ng; ++j) s += Tb[j * ng + ii] * xs[bo + j];
    }
    ts[i] = s;
  }
  __syncthreads();
  lus::lu_solve<1, false>(LU + soff[b], n, ts, tmp, nullptr);
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int k = pos2k[v0 + i];
    const int bo = sub_glob_boff[k], ng = gsize[sub_globs[k]];
    const double* Tb = TT + sh_doff[sub_glob_sh[k]] + (long long)(i - bo) * ng;
    double s = 0.0;
    for (int j = 0; j < ng; ++j) s += Tb[j] * ts[bo + j];
    y[v0 + i] = s;
  }
}

// Primal pieces through the LU, one CTA per subdomain, 8 (n_p <= 8) or 16
// primal columns at a time (every sweep reads the whole LU once: the kernel is
// bound by that traffic, so as many right-hand sides as fit share a sweep):
//   MP[p] = e_pc - Z Sbar[:, pc],  RP[p] = e_pc - Z^T Sbar[pc, :]^T,  C_i[p][q] = Sbar[pr, :] . MP[q]
// (Z = Sdd^-1 embedded with zero primal rows / columns)
constexpr int kPL = 16;

template <int NR>
BDDC_DEV void primal_pieces_chunk(int n, int c0, int pc_n, const unsigned char* pm,
                                  const int* __restrict__ ppos_b, const double* __restrict__ Sr,
                                  const double* __restrict__ Sc, const double* __restrict__ L,
                                  double* __restrict__ Mb, double* __restrict__ Rb, double* X,
                                  double* tmp) {
  constexpr int XS = lus::xstride<NR>();
  for (int idx = threadIdx.x; idx < n * NR; idx += blockDim.x) {
    const int q = idx / n, r = idx - q * n;  // coalesced along the Sbar column (stored as a row)
    X[r * XS + q] = (q < pc_n && !pm[r]) ? Sc[(long long)(c0 + q) * n + r] : 0.0;
  }
  __syncthreads();
  lus::lu_solve<NR, false>(L, n, X, tmp, nullptr);
  for (int idx = threadIdx.x; idx < n * pc_n; idx += blockDim.x) {
    const int q = idx / n, r = idx - q * n;
    Mb[(long long)(c0 + q) * n + r] = (r == ppos_b[c0 + q] ? 1.0 : 0.0) - X[r * XS + q];
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < n * NR; idx += blockDim.x) {
    const int q = idx / n, r = idx - q * n;  // coalesced along the Sbar row
    X[r * XS + q] = (q < pc_n && !pm[r]) ? Sr[(long long)(c0 + q) * n + r] : 0.0;
  }
  __syncthreads();
  lus::lu_solve<NR, true>(L, n, X, tmp, nullptr);
  for (int idx = threadIdx.x; idx < n * pc_n; idx += blockDim.x) {
    const int q = idx / n, r = idx - q * n;
    Rb[(long long)(c0 + q) * n + r] = (r == ppos_b[c0 + q] ? 1.0 : 0.0) - X[r * XS + q];
  }
  __syncthreads();
}

__global__ void __launch_bounds__(256, 3) primal_pieces_lu_kernel(
    const int* __restrict__ nB, const long long* __restrict__ soff,
    const long long* __restrict__ voff, const unsigned char* __restrict__ primal_mask,
    const int* __restrict__ pstart, const int* __restrict__ ppos,
    const long long* __restrict__ poff, const double* __restrict__ Srows,
    const double* __restrict__ Scols, const double* __restrict__ LU, double* __restrict__ MP,
    double* __restrict__ RP, double* __restrict__ Cl, const long long* __restrict__ coff) {
  extern __shared__ double psm[];
  const int b = blockIdx.x;
  const int n = nB[b];
  const int p0 = pstart[b], np = pstart[b + 1] - p0;
  if (np == 0) return;
  double* X = psm;                                  // n x xstride
  double* tmp = psm + n * lus::xstride<kPL>();      // 64 x xstride
  const double* Sr = Srows + poff[b];  // Sbar[ppos_q, :] as row q (n_p x n)
  const double* Sc = Scols + poff[b];  // Sbar[:, ppos_q] as row q
  const double* L = LU + soff[b];
  const unsigned char* pm = primal_mask + voff[b];
  double* Mb = MP + poff[b];
  double* Rb = RP + poff[b];
  if (np <= 8) {
    primal_pieces_chunk<8>(n, 0, np, pm, ppos + p0, Sr, Sc, L, Mb, Rb, X, tmp);
  } else {
    for (int c0 = 0; c0 < np; c0 += kPL) {
      const int left = np - c0;
      if (left <= 8) primal_pieces_chunk<8>(n, c0, left, pm, ppos + p0, Sr, Sc, L, Mb, Rb, X, tmp);
      else primal_pieces_chunk<kPL>(n, c0, min(kPL, left), pm, ppos + p0, Sr, Sc, L, Mb, Rb, X, tmp);
    }
  }
  double* C = Cl + coff[b];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int i = warp; i < np * np; i += nw) {
    const int p = i / np, q = i - p * np;
    double v = 0.0;
    for (int k = lane; k < n; k += 32) v += Sr[(long long)p * n + k] * Mb[(long long)q * n + k];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) C[i] = v;
  }
}

// rows form: Out[p][c] = sum over block of c: In[p][bo+q] * TT-derived value
//   G = RP T   where T = Q D^T blockdiag: G[p][c] = sum_q RP[p][bo+q] T[bo+q][c]
//            T[bo+q][c] = TT^T block [q][c-bo]  = TTb[(c-bo)*ng + q]
//   Nt = (T^T MP^T)^T = MP T : same form as G with In = MP
__global__ void primal_rows_times_T_kernel(SubGlobMap m, const double* __restrict__ TT,
                                           const int* __restrict__ pstart,
                                           const long long* __restrict__ poff,
                                           const double* __restrict__ In,
                                           double* __restrict__ Out) {
  const int b = blockIdx.y;
  const int n = m.nB[b];
  const int np = pstart[b + 1] - pstart[b];
  const double* X = In + poff[b];
  double* Y = Out + poff[b];
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < (long long)np * n;
       idx += (long long)gridDim.x * blockDim.x) {
    const int p = (int)(idx / n), c = (int)(idx - (long long)p * n);
    const int k = m.pos2k[m.voff[b] + c];
    const int bo = m.sub_glob_boff[k];
    const int ng = m.gsize[m.sub_globs[k]];
    const double* Tb = TT + m.sh_doff[m.sub_glob_sh[k]];
    const int cc = c - bo;
    double s = 0.0;
    for (int q = 0; q < ng; ++q) s += X[(long long)p * n + bo + q] * Tb[cc * ng + q];
    Y[idx] = s;
  }
}

// coarse assembly C[gp][gq] = sum_i C_i[p][q], deterministic: one warp owns
// coarse row gp, zeroes it, then adds the rows of its sources (the (subdomain,
// local primal) pairs mapped to gp, csrc[cstart[gp]..cstart[gp+1]) in ascending
// subdomain order) one after the other; within one source the columns
// pgid[p0 + q] are distinct, so the lanes never collide.
__global__ void coarse_scatter_kernel(const int* __restrict__ pstart, const int* __restrict__ pgid,
                                      const double* __restrict__ Cl,
                                      const long long* __restrict__ coff,
                                      const long long* __restrict__ cstart,
                                      const long long* __restrict__ csrc, double* __restrict__ C,
                                      long long ldc, int n_c, int nbatch) {
  const int gp = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (gp >= n_c) return;
  double* row = C + (long long)gp * ldc;
  for (int c = lane; c < n_c; c += 32) row[c] = 0.0;
  __syncwarp();
  for (long long s = cstart[gp]; s < cstart[gp + 1]; ++s) {
    const int f = (int)csrc[s];
    int lo = 0, hi = nbatch;  // largest b with pstart[b] <= f
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (pstart[mid] <= f) lo = mid; else hi = mid;
    }
    const int b = lo, p0 = pstart[b], np = pstart[b + 1] - p0, p = f - p0;
    const double* Cb = Cl + coff[b] + (long long)p * np;
    for (int q = lane; q < np; q += 32) row[pgid[p0 + q]] += Cb[q];
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// batched GEMV families for the apply
// ---------------------------------------------------------------------------
// y_i = S_i x_i with x_i = u[perm_i]; y written to the local buffer (voff)
// One CTA per (subdomain, row chunk); x staged in shared memory.
template <bool ACCUM_PRIMAL>
__global__ void __launch_bounds__(256) local_gemv_kernel(
    const int* __restrict__ nB, const long long* __restrict__ soff,
    const long long* __restrict__ voff, const int* __restrict__ iface_perm,
    const double* __restrict__ Mat, const double* __restrict__ u, double* __restrict__ y,
    // primal restriction (only when ACCUM_PRIMAL): c = G x
    const int* __restrict__ pstart, const long long* __restrict__ poff,
    const double* __restrict__ G, double* __restrict__ cvals) {
  extern __shared__ double xs[];
  const int b = blockIdx.y;
  const int n = nB[b];
  const int chunk = (n + gridDim.x - 1) / gridDim.x;
  const int r0 = blockIdx.x * chunk;
  const int* pm = iface_perm + voff[b];
  for (int j = threadIdx.x; j < n; j += blockDim.x) xs[j] = u[pm[j]];
  __syncthreads();
  const double* A = Mat + soff[b];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int r1 = min(n, r0 + chunk);
  for (int r = r0 + warp; r < r1; r += nw) {
    const double* row = A + (long long)r * n;
    double s = 0.0;
    for (int c = lane; c < n; c += 32) s += row[c] * xs[c];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) y[voff[b] + r] = s;
  }
  if (ACCUM_PRIMAL && blockIdx.x == 0) {
    const int np = pstart[b + 1] - pstart[b];
    const double* Gb = G + poff[b];
    for (int p = warp; p < np; p += nw) {
      const double* row = Gb + (long long)p * n;
      double s = 0.0;
      for (int c = lane; c < n; c += 32) s += row[c] * xs[c];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) cvals[pstart[b] + p] = s;
    }
  }
}

// y_i += sum_p Nt_i[p, :] * uP[pgid_i[p]]
__global__ void prolong_primal_kernel(const int* __restrict__ nB, const long long* __restrict__ voff,
                                      const int* __restrict__ pstart, const int* __restrict__ pgid,
                                      const long long* __restrict__ poff,
                                      const double* __restrict__ Nt, const double* __restrict__ uP,
                                      double* __restrict__ y) {
  const int b = blockIdx.y;
  const int n = nB[b];
  const int p0 = pstart[b], np = pstart[b + 1] - p0;
  const double* Nb = Nt + poff[b];
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int p = 0; p < np; ++p) s += Nb[(long long)p * n + r] * uP[pgid[p0 + p]];
    y[voff[b] + r] += s;
  }
}

// deterministic gather-reduce: out[t] = sum_{j in src(t)} y[src[j]]  (CSR, sorted by subdomain)
__global__ void gather_reduce_kernel(const long long* __restrict__ tstart,
                                     const long long* __restrict__ tsrc,
                                     const double* __restrict__ y, double* __restrict__ out,
                                     long long n) {
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (long long)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (long long j = tstart[t]; j < tstart[t + 1]; ++j) s += y[tsrc[j]];
    out[t] = s;
  }
}

// ---------------------------------------------------------------------------
// coarse triangular solves with the blocked no-pivot LU from schur_eliminate
//   forward:  t_k = P_k b_k ; b_i -= A[i, k:k+w] t_k  (i >= k+w)
//   backward: x_k = t_k     ; t_i -= A[i, k:k+w] x_k  (i < k)
// ---------------------------------------------------------------------------
// Coarse envelope solve in one cooperative persistent kernel (grid-wide
// barrier per 64-wide panel instead of a kernel launch):
//   forward  b_i -= L'_ik b_k            i in [k+w, lim_k)
//   t = blockdiag(P_k) b
//   backward t_i -= W_ik x_k (x_k = t_k)  i in [first_k, k)
#ifndef BDDC_COOP_THREADS
#define BDDC_COOP_THREADS 256
#endif
#ifndef BDDC_COOP_CTAS
#define BDDC_COOP_CTAS 0   // 0: one CTA per SM
#endif

__global__ void __launch_bounds__(BDDC_COOP_THREADS) coarse_solve_coop_kernel(
    const double* __restrict__ A, long long ld, int n, const double* __restrict__ pinv,
    long long pstride, const int* __restrict__ lim, const int* __restrict__ first,
    double* __restrict__ b, double* __restrict__ t) {
  cg::grid_group grid = cg::this_grid();
  const int nP = (n + 63) / 64;
  const int lane = threadIdx.x & 31;
  const int gw = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int nwarps = (int)((gridDim.x * blockDim.x) >> 5);
  for (int p = 0; p < nP; ++p) {
    const int k = p * 64, w = min(64, n - k), L = min(n, lim[p]);
    if (p > 0) grid.sync();
    if (k + w >= L) continue;
    const double b0 = lane < w ? b[k + lane] : 0.0;
    const double b1 = lane + 32 < w ? b[k + lane + 32] : 0.0;
    for (int i = k + w + gw; i < L; i += nwarps) {
      const double* row = A + (long long)i * ld + k;
      double s = (lane < w ? row[lane] * b0 : 0.0) + (lane + 32 < w ? row[lane + 32] * b1 : 0.0);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) b[i] -= s;
    }
  }
  grid.sync();
  for (int r = gw; r < n; r += nwarps) {
    const int p = r >> 6, k = p * 64, w = min(64, n - k);
    const double* Pr = pinv + (long long)p * pstride + (r - k) * 64;
    double s = (lane < w ? Pr[lane] * b[k + lane] : 0.0) +
               (lane + 32 < w ? Pr[lane + 32] * b[k + lane + 32] : 0.0);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) t[r] = s;
  }
  for (int p = nP - 1; p >= 1; --p) {
    const int k = p * 64, w = min(64, n - k), F = max(0, first[p]);
    grid.sync();
    if (F >= k) continue;
    const double x0 = lane < w ? t[k + lane] : 0.0;
    const double x1 = lane + 32 < w ? t[k + lane + 32] : 0.0;
    for (int i = F + gw; i < k; i += nwarps) {
      const double* row = A + (long long)i * ld + k;
      double s = (lane < w ? row[lane] * x0 : 0.0) + (lane + 32 < w ? row[lane + 32] * x1 : 0.0);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) t[i] -= s;
    }
  }
}

// ---------------------------------------------------------------------------
// Coarse envelope solve as a dataflow over 128-row super-panels: CTA c owns
// super-panels Q = c, c + grid, ...; a super-panel's rows are final once the
// super-panels it depends on have published theirs (flag == epoch), so the
// only serial chain is "flag -> 128x128 block GEMV -> flag" instead of one
// grid-wide barrier per 64-wide panel.  The block on the critical path (the
// neighbouring super-panel) is prefetched into shared memory with cp.async
// while the older contributions are applied.
//   forward:  b_Q -= sum_{J<Q} L'[Q, J] b_J ; then within Q: b_hi -= L'[hi, lo] b_lo
//             t_Q = blockdiag(P) b_Q
//   backward: x_Q = t_Q - sum_{J>Q} W[Q, J] x_J ; then x_lo -= W[lo, hi] x_hi
// ---------------------------------------------------------------------------
constexpr int kSP = 128;

BDDC_DEV int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
BDDC_DEV void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

BDDC_DEV void wait_flag(const int* f, int epoch) {
  if (threadIdx.x == 0) {
    while (ld_acquire(f) != epoch) __nanosleep(32);
  }
  __syncthreads();
}

// acc[r] -= sum_c blk[r][c] v[c]   (r < h, c < w <= 128); warp per 4 rows (16 loads in
// flight per lane when blk is in global memory)
BDDC_DEV void block_gemv_sub(const double* blk, long long ldb, int h, int w, const double* v,
                             double* acc) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  double vv[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) vv[j] = (lane + 32 * j < w) ? v[lane + 32 * j] : 0.0;
  for (int r0 = 4 * warp; r0 < h; r0 += 4 * nw) {
    double s[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      s[i] = 0.0;
      if (r0 + i < h) {
        const double* row = blk + (long long)(r0 + i) * ldb;
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (lane + 32 * j < w) s[i] = fma(row[lane + 32 * j], vv[j], s[i]);
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s[i] += __shfl_xor_sync(0xffffffffu, s[i], o);
    if (lane < 4 && r0 + lane < h) {
      double x = s[0];
#pragma unroll
      for (int i = 1; i < 4; ++i)
        if (lane == i) x = s[i];
      acc[r0 + lane] -= x;
    }
  }
}

__global__ void __launch_bounds__(256, 1) coarse_solve_flow_kernel(
    const double* __restrict__ A, long long ld, int n, const double* __restrict__ pinv,
    long long pstride, const int* __restrict__ jmin, const int* __restrict__ jmax,
    double* __restrict__ b, double* __restrict__ t, int* __restrict__ flags, int epoch) {
  extern __shared__ __align__(16) double fsm[];
  double* buf = fsm;                 // kSP x kSP prefetched block (neighbour super-panel)
  double* dg = buf + kSP * kSP;      // 64 x 64 prefetched intra-super-panel block
  double* acc = dg + 64 * 64;        // kSP
  double* v = acc + kSP;             // kSP
  const int nQ = (n + kSP - 1) / kSP;
  int* fflag = flags;
  int* bflag = flags + nQ;
  // ---- forward + diagonal ----
  for (int Q = blockIdx.x; Q < nQ; Q += gridDim.x) {
    const int r0 = Q * kSP, h = min(kSP, n - r0);
    const int Jlo = jmin[Q];
    const bool pre = Q - 1 >= Jlo;
    if (h > 64) {
      const double* src = A + (long long)(r0 + 64) * ld + r0;
      for (int idx = threadIdx.x; idx < (h - 64) * 64; idx += blockDim.x) {
        const int r = idx >> 6, c = idx & 63;
        cp_async8(dg + idx, src + (long long)r * ld + c, true);
      }
    }
    if (pre) {
      const double* src = A + (long long)r0 * ld + (Q - 1) * kSP;
      for (int idx = threadIdx.x; idx < h * kSP; idx += blockDim.x) {
        const int r = idx / kSP, c = idx - r * kSP;
        cp_async8(buf + idx, src + (long long)r * ld + c, true);
      }
    }
    cp_async_commit();
    for (int i = threadIdx.x; i < h; i += blockDim.x) acc[i] = b[r0 + i];
    __syncthreads();
    for (int J = Jlo; J < Q - 1; ++J) {
      wait_flag(fflag + J, epoch);
      for (int i = threadIdx.x; i < kSP; i += blockDim.x) v[i] = __ldcg(b + J * kSP + i);
      __syncthreads();
      block_gemv_sub(A + (long long)r0 * ld + J * kSP, ld, h, kSP, v, acc);
      __syncthreads();
    }
    if (pre) {
      wait_flag(fflag + Q - 1, epoch);
      for (int i = threadIdx.x; i < kSP; i += blockDim.x) v[i] = __ldcg(b + (Q - 1) * kSP + i);
      cp_async_wait<0>();
      __syncthreads();
      block_gemv_sub(buf, kSP, h, kSP, v, acc);
      __syncthreads();
    }
    cp_async_wait<0>();
    __syncthreads();
    if (h > 64) {  // lower half of the super-panel from its upper half
      block_gemv_sub(dg, 64, h - 64, 64, acc, acc + 64);
      __syncthreads();
    }
    for (int i = threadIdx.x; i < h; i += blockDim.x) b[r0 + i] = acc[i];
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      st_release(fflag + Q, epoch);
    }
    // t = blockdiag(P_p) b for the two 64-panels (v = 0 - P b, then negated)
    for (int i = threadIdx.x; i < kSP; i += blockDim.x) v[i] = 0.0;
    __syncthreads();
    for (int hp = 0; hp * 64 < h; ++hp) {
      const int w = min(64, h - hp * 64);
      block_gemv_sub(pinv + (long long)(2 * Q + hp) * pstride, 64, w, w, acc + hp * 64, v + hp * 64);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < h; i += blockDim.x) t[r0 + i] = -v[i];
    __syncthreads();
  }
  // ---- backward ----
  const int qlast = blockIdx.x + ((nQ - 1 - (int)blockIdx.x) / (int)gridDim.x) * (int)gridDim.x;
  for (int Q = qlast; Q >= 0 && Q < nQ; Q -= gridDim.x) {
    const int r0 = Q * kSP, h = min(kSP, n - r0);
    const int Jhi = jmax[Q];
    const bool pre = Q + 1 <= Jhi;
    if (h > 64) {
      const double* src = A + (long long)r0 * ld + r0 + 64;
      for (int idx = threadIdx.x; idx < 64 * 64; idx += blockDim.x) {
        const int r = idx >> 6, c = idx & 63;
        cp_async8(dg + idx, c < h - 64 ? src + (long long)r * ld + c : src, c < h - 64);
      }
    }
    if (pre) {
      const int w = min(kSP, n - (Q + 1) * kSP);
      const double* src = A + (long long)r0 * ld + (Q + 1) * kSP;
      for (int idx = threadIdx.x; idx < h * kSP; idx += blockDim.x) {
        const int r = idx / kSP, c = idx - r * kSP;
        cp_async8(buf + idx, c < w ? src + (long long)r * ld + c : src, c < w);
      }
    }
    cp_async_commit();
    for (int i = threadIdx.x; i < h; i += blockDim.x) acc[i] = t[r0 + i];
    __syncthreads();
    for (int J = Jhi; J > Q + 1; --J) {
      const int w = min(kSP, n - J * kSP);
      wait_flag(bflag + J, epoch);
      for (int i = threadIdx.x; i < w; i += blockDim.x) v[i] = __ldcg(t + J * kSP + i);
      __syncthreads();
      block_gemv_sub(A + (long long)r0 * ld + J * kSP, ld, h, w, v, acc);
      __syncthreads();
    }
    if (pre) {
      const int w = min(kSP, n - (Q + 1) * kSP);
      wait_flag(bflag + Q + 1, epoch);
      for (int i = threadIdx.x; i < w; i += blockDim.x) v[i] = __ldcg(t + (Q + 1) * kSP + i);
      cp_async_wait<0>();
      __syncthreads();
      block_gemv_sub(buf, kSP, h, w, v, acc);
      __syncthreads();
    }
    cp_async_wait<0>();
    __syncthreads();
    if (h > 64) {  // upper half from the (final) lower half
      block_gemv_sub(dg, 64, 64, h - 64, acc + 64, acc);
      __syncthreads();
    }
    for (int i = threadIdx.x; i < h; i += blockDim.x) t[r0 + i] = acc[i];
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      st_release(bflag + Q, epoch);
    }
  }
}

}  // namespace bddc

// ===========================================================================
// C-ABI
// ===========================================================================
using namespace bddc;

static int pc_status() {
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : -(int)e;
}

static SubGlobMap make_map(const int* nB, const long long* soff, const long long* voff,
                           const int* pos2k, const int* sub_globs, const int* sub_glob_boff,
                           const int* sub_glob_sh, const int* gsize, const double* Q,
                           const long long* q_off, const double* D, const long long* sh_doff) {
  SubGlobMap m;
  m.nB = nB; m.soff = soff; m.voff = voff; m.pos2k = pos2k; m.sub_globs = sub_globs;
  m.sub_glob_boff = sub_glob_boff; m.sub_glob_sh = sub_glob_sh; m.gsize = gsize; m.Q = Q;
  m.q_off = q_off; m.D = D; m.sh_doff = sh_doff;
  return m;
}

extern "C" {

static int glob_block_smem(int max_ng) {
  return (64 * 64 + (max_ng > kBT_COLS ? max_ng : kBT_COLS) * kBT_COLS) * (int)sizeof(double);
}

constexpr int kMmaMinNg = 16;  // smaller glob blocks: per-element kernel

static int glob_mma(const int* nB, const long long* soff, const int* sub_glob_start, int nsub,
                    const int* sub_globs, const int* sub_glob_boff, const int* sub_glob_sh,
                    const int* gsize, const double* L, const double* LT, const long long* loff,
                    int by_slot, int right, const double* in, double* out, int n_items,
                    int max_nB, int max_ng, int max_globs, cudaStream_t stream) {
  static PerDeviceOnce once;
  once([&] {
    cudaFuncSetAttribute(glob_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(TileSmem));
  });
  if (max_ng >= kMmaMinNg) {
    const int tpi = ceil_div(max_nB, 64);
    dim3 grid((unsigned)(n_items * tpi), ceil_div(max_ng, 64));
    glob_mma_kernel<<<grid, kTileThreads, sizeof(TileSmem), stream>>>(
        nB, soff, sub_glob_start, nsub, sub_globs, sub_glob_boff, sub_glob_sh, gsize, L, LT, loff,
        by_slot, right, in, out, tpi, kMmaMinNg);
    bddc_note_launches(1);
  }
  // small blocks (vertices, short edges): per-element kernel, L from Q (by glob) or TT (by slot)
  SubGlobMap m;
  m.nB = nB; m.soff = soff; m.voff = nullptr; m.pos2k = nullptr; m.sub_globs = sub_globs;
  m.sub_glob_boff = sub_glob_boff; m.sub_glob_sh = sub_glob_sh; m.gsize = gsize;
  m.Q = by_slot ? nullptr : L; m.q_off = by_slot ? nullptr : loff; m.D = nullptr;
  m.sh_doff = by_slot ? loff : nullptr;
  const int smem = (64 * 64 + 32 * 32) * (int)sizeof(double);
  glob_block_kernel<<<dim3(max_globs, nsub), 256, smem, stream>>>(
      m, sub_glob_start, by_slot ? L : nullptr, in, out, by_slot ? 1 : 0, right, 16, kMmaMinNg);
  bddc_note_launches(1);
  return pc_status();
}

// Sbar = Qi S Qi^T (via tmp); QT: caller scratch of the Q buffer's size
int bddc_pc_transform_schur(const int* nB, const long long* soff, const int* sub_glob_start,
                            int nbatch, const int* sub_globs, const int* sub_glob_boff,
                            const int* sub_glob_sh, const int* gsize, const double* Q,
                            const long long* q_off, double* QT, int n_globs, int n_items,
                            int max_nB, int max_ng, int max_globs, const double* S, double* tmp,
                            double* Sbar, cudaStream_t stream) {
  if (nbatch <= 0) return 0;
  transpose_blocks_kernel<<<n_globs, 128, 0, stream>>>(Q, QT, q_off, nullptr, gsize, n_globs);
  bddc_note_launches(1);
  int st = glob_mma(nB, soff, sub_glob_start, nbatch, sub_globs, sub_glob_boff, sub_glob_sh, gsize,
                    Q, QT, q_off, 0, 0, S, tmp, n_items, max_nB, max_ng, max_globs, stream);
  if (st) return st;
  return glob_mma(nB, soff, sub_glob_start, nbatch, sub_globs, sub_glob_boff, sub_glob_sh, gsize,
                  Q, QT, q_off, 0, 1, tmp, Sbar, n_items, max_nB, max_ng, max_globs, stream);
}

int bddc_pc_glob_reflectors(const int* kind, const int* gsize, const int* r, double* Q,
                            const long long* q_off, double* HV, double* W, const long long* w_off,
                            int n_globs, int max_ng, cudaStream_t stream) {
  if (n_globs <= 0) return 0;
  glob_reflectors_kernel<<<n_globs, 128, (max_ng + 4) * (int)sizeof(double), stream>>>(
      kind, gsize, r, Q, q_off, HV, W, w_off);
  bddc_note_launches(1);
  return pc_status();
}

int bddc_pc_transform_refl(const int* nB, const long long* soff, const int* sub_glob_start,
                           const int* sub_globs, const int* sub_glob_boff, const int* kind,
                           const int* gsize, const int* r, const double* HV,
                           const long long* q_off, const double* S, double* Sbar, int nbatch,
                           cudaStream_t stream) {
  if (nbatch <= 0) return 0;
  transform_refl_kernel<<<nbatch, 256, 0, stream>>>(nB, soff, sub_glob_start, sub_globs,
                                                    sub_glob_boff, kind, gsize, r, HV, q_off, S,
                                                    Sbar);
  bddc_note_launches(1);
  return pc_status();
}

int bddc_pc_ttblocks(const int* slot_glob, const int* gsize, const double* Q,
                     const long long* q_off, const double* D, const long long* sh_doff,
                     double* TT, int n_slots, cudaStream_t stream) {
  if (n_slots <= 0) return 0;
  ttblock_kernel<<<n_slots, 128, 0, stream>>>(slot_glob, gsize, Q, q_off, D, sh_doff, TT, n_slots); bddc_note_launches(1);
  return pc_status();
}

int bddc_pc_dbar(const int* slot_glob, const int* slot_sub, const int* gsize, const int* sh_boff,
                 const long long* sh_doff, const double* Q, const long long* q_off,
                 const double* TT, const int* nB, const long long* soff, const long long* voff,
                 const int* nodal, double* W, double* Dbar, int n_slots, cudaStream_t stream) {
  if (n_slots <= 0) return 0;
  dbar_kernel<<<n_slots, 128, 0, stream>>>(slot_glob, slot_sub, gsize, sh_boff, sh_doff, Q, q_off,
                                           TT, nB, soff, voff, nodal, W, Dbar);
  bddc_note_launches(1);
  return pc_status();
}

int bddc_transpose_batched(const double* X, const long long* soff, const int* n, int nbatch,
                           double* out, cudaStream_t stream) {
  if (nbatch <= 0) return 0;
  transpose_batched_kernel<<<dim3(32, nbatch), 256, 0, stream>>>(X, soff, n, out);
  bddc_note_launches(1);
  return pc_status();
}

int bddc_pc_dual_embed(const int* nB, const long long* soff, const long long* voff,
                       const unsigned char* primal_mask, const double* Sbar, double* Zin,
                       double* Csym, int nbatch, cudaStream_t stream) {
  if (nbatch <= 0) return 0;
  dual_embed_kernel<<<dim3(64, nbatch), 256, 0, stream>>>(nB, soff, voff, primal_mask, Sbar, Zin,
                                                          Csym); bddc_note_launches(1);
  return pc_status();
}




int bddc_pc_primal_rows_T(const int* nB, const long long* voff, const int* pos2k,
                          const int* sub_globs, const int* sub_glob_boff, const int* sub_glob_sh,
                          const int* gsize, const long long* sh_doff, const double* TT,
                          const int* pstart, const long long* poff, const double* In, double* Out,
                          int nbatch, cudaStream_t stream) {
  if (nbatch <= 0) return 0;
  SubGlobMap m = make_map(nB, nullptr, voff, pos2k, sub_globs, sub_glob_boff, sub_glob_sh, gsize,
                          nullptr, nullptr, nullptr, sh_doff);
  primal_rows_times_T_kernel<<<dim3(16, nbatch), 256, 0, stream>>>(m, TT, pstart, poff, In, Out); bddc_note_launches(1);
  return pc_status();
}

int bddc_lu_diag_pinv(double* LU, const long long* soff, const int* nB, int nbatch, int max_n,
                      const double* pinv, long long pinv_stride, long long step_stride,
                      cudaStream_t stream) {
  if (nbatch <= 0 || max_n <= 0) return 0;
  lu_diag_pinv_kernel<<<dim3(ceil_div(max_n, 64), nbatch), 256, 0, stream>>>(LU, soff, nB, pinv,
                                                                             pinv_stride, step_stride);
  bddc_note_launches(1);
  return pc_status();
}

int bddc_pc_local_solve(const int* nB, const long long* soff, const long long* voff,
                        const int* iface_perm, const double* LU, const int* pos2k,
                        const int* sub_globs, const int* sub_glob_boff, const int* sub_glob_sh,
                        const int* gsize, const long long* sh_doff, const double* TT,
                        const unsigned char* primal_mask, const double* u, double* y,
                        const int* pstart, const long long* poff, const double* G, double* cvals,
                        int nbatch, int max_nB, cudaStream_t stream) {
  if (nbatch <= 0) return 0;
  const int smem = (2 * max_nB + 64) * (int)sizeof(double);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(local_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  local_solve_kernel<<<nbatch, 256, smem, stream>>>(nB, soff, voff, iface_perm, LU, pos2k, sub_globs,
                                                    sub_glob_boff, sub_glob_sh, gsize, sh_doff, TT,
                                                    primal_mask, u, y, pstart, poff, G, cvals);
  bddc_note_launches(1);
  return pc_status();
}

int bddc_pc_primal_restrict(const int* nB, const long long* voff, const int* iface_perm,
                            const double* u, const int* pstart, const long long* poff,
                            const double* G, double* cvals, int nbatch, int max_nB,
                            cudaStream_t stream) {
  if (nbatch <= 0) return 0;
  const int smem = max_nB * (int)sizeof(double);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(primal_restrict_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  primal_restrict_kernel<<<nbatch, 256, smem, stream>>>(nB, voff, iface_perm, u, pstart, poff, G,
                                                        cvals);
  bddc_note_launches(1);
  return pc_status();
}

int bddc_pc_transform_embed(const int* nB, const long long* soff, const long long* voff,
                            const int* pos2k, const int* sub_globs, const int* sub_glob_boff,
                            const int* kind, const int* gsize, const int* r, const double* HV,
                            const long long* q_off, const int* refl_start, const int* refl_k,
                            const int* left_k, const int* left_sub, int n_left, const int* pidx,
                            const long long* poff, const double* S, double* Z, double* Srows,
                            double* Scols, int nbatch, int max_nB, cudaStream_t stream) {
  if (nbatch <= 0) return 0;
  if (n_left > 0) {
    transform_left_kernel<<<n_left, 256, 0, stream>>>(nB, soff, left_k, left_sub, sub_globs,
                                                      sub_glob_boff, gsize, r, HV, q_off, S, Z);
    bddc_note_launches(1);
  }
  const int smem = 8 * max_nB * (int)sizeof(double);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(transform_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  transform_rows_kernel<<<dim3(ceil_div(max_nB, 8), nbatch), 256, smem, stream>>>(
      nB, soff, voff, pos2k, sub_globs, sub_glob_boff, kind, gsize, r, HV, q_off, refl_start,
      refl_k, pidx, poff, S, Z, Srows, Scols, max_nB);
  bddc_note_launches(1);
  return pc_status();
}

int bddc_pc_primal_extract(const int* nB, const long long* soff, const long long* voff,
                           const int* pidx, const long long* poff, const double* Sbar,
                           double* Srows, double* Scols, int nbatch, cudaStream_t stream) {
  if (nbatch <= 0) return 0;
  primal_extract_kernel<<<dim3(64, nbatch), 256, 0, stream>>>(nB, soff, voff, pidx, poff, Sbar,
                                                              Srows, Scols);
  bddc_note_launches(1);
  return pc_status();
}

int bddc_pc_primal_pieces_lu(const int* nB, const long long* soff, const long long* voff,
                             const unsigned char* primal_mask, const int* pstart, const int* ppos,
                             const long long* poff, const double* Srows, const double* Scols,
                             const double* LU, double* MP, double* RP, double* Cl,
                             const long long* coff, int nbatch, int max_nB, cudaStream_t stream) {
  if (nbatch <= 0) return 0;
  const int smem = (max_nB * lus::xstride<kPL>() + 64 * lus::xstride<kPL>()) * (int)sizeof(double);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(primal_pieces_lu_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  primal_pieces_lu_kernel<<<nbatch, 256, smem, stream>>>(nB, soff, voff, primal_mask, pstart, ppos,
                                                         poff, Srows, Scols, LU, MP, RP, Cl, coff);
  bddc_note_launches(1);
  return pc_status();
}

int bddc_coarse_scatter(const int* pstart, const int* pgid, const double* Cl,
                        const long long* coff, const long long* cstart, const long long* csrc,
                        double* C, long long ldc, int n_c, int nbatch, cudaStream_t stream) {
  if (n_c <= 0) return 0;
  coarse_scatter_kernel<<<ceil_div(n_c, 8), 256, 0, stream>>>(pstart, pgid, Cl, coff, cstart, csrc,
                                                             C, ldc, n_c, nbatch);
  bddc_note_launches(1);
  return pc_status();
}

int bddc_local_gemv(const int* nB, const long long* soff, const long long* voff,
                    const int* iface_perm, const double* M, const double* u, double* y,
                    const int* pstart, const long long* poff, const double* G, double* cvals,
                    int nbatch, int max_nB, int row_chunks, cudaStream_t stream) {
  if (nbatch <= 0) return 0;
  const int smem = max_nB * (int)sizeof(double);
  if (G) {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(local_gemv_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    local_gemv_kernel<true><<<dim3(row_chunks, nbatch), 256, smem, stream>>>(
        nB, soff, voff, iface_perm, M, u, y, pstart, poff, G, cvals); bddc_note_launches(1);
  } else {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(local_gemv_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    local_gemv_kernel<false><<<dim3(row_chunks, nbatch), 256, smem, stream>>>(
        nB, soff, voff, iface_perm, M, u, y, nullptr, nullptr, nullptr, nullptr); bddc_note_launches(1);
  }
  return pc_status();
}

int bddc_prolong_primal(const int* nB, const long long* voff, const int* pstart, const int* pgid,
                        const long long* poff, const double* Nt, const double* uP, double* y,
                        int nbatch, cudaStream_t stream) {
  if (nbatch <= 0) return 0;
  prolong_primal_kernel<<<dim3(2, nbatch), 256, 0, stream>>>(nB, voff, pstart, pgid, poff, Nt, uP, y); bddc_note_launches(1);
  return pc_status();
}

int bddc_gather_reduce(const long long* tstart, const long long* tsrc, const double* y,
                       double* out, long long n, cudaStream_t stream) {
  if (n <= 0) return 0;
  gather_reduce_kernel<<<ceil_div(n, 256), 256, 0, stream>>>(tstart, tsrc, y, out, n); bddc_note_launches(1);
  return pc_status();
}

int bddc_coarse_solve(const double* A, long long ld, int n, const double* pinv,
                      long long pinv_step_stride, const int* lim, const int* first, double* b,
                      double* t, cudaStream_t stream) {
  if (n <= 0) return 0;
  static PerDeviceInt cached;
  const int grid = cached.get([] {
    int dev = current_device(), sms = 0, per_sm = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, coarse_solve_coop_kernel,
                                                  BDDC_COOP_THREADS, 0);
    int g = BDDC_COOP_CTAS > 0 ? BDDC_COOP_CTAS : sms;
    if (g > sms * per_sm) g = sms * per_sm;
    return g <= 0 ? 1 : g;
  });
  void* args[] = {(void*)&A, (void*)&ld, (void*)&n, (void*)&pinv, (void*)&pinv_step_stride,
                  (void*)&lim, (void*)&first, (void*)&b, (void*)&t};
  cudaError_t e = cudaLaunchCooperativeKernel((const void*)coarse_solve_coop_kernel, dim3(grid),
                                              dim3(BDDC_COOP_THREADS), args, 0, stream);
  bddc_note_launches(1);
  return e == cudaSuccess ? pc_status() : -(int)e;
}

int bddc_coarse_solve_flow(const double* A, long long ld, int n, const double* pinv,
                           long long pinv_step_stride, const int* jmin, const int* jmax, double* b,
                           double* t, int* flags, int epoch, cudaStream_t stream) {
  if (n <= 0) return 0;
  const int smem = (kSP * kSP + 64 * 64 + 2 * kSP) * (int)sizeof(double);
  static PerDeviceInt cached;
  const int grid = cached.get([smem] {
    int dev = current_device(), sms = 0, per_sm = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(coarse_solve_flow_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, coarse_solve_flow_kernel, 256, smem);
    return sms * (per_sm > 0 ? per_sm : 1);
  });
  const int nQ = (n + kSP - 1) / kSP;
  int g = nQ < grid ? nQ : grid;
  void* args[] = {(void*)&A, (void*)&ld, (void*)&n, (void*)&pinv, (void*)&pinv_step_stride,
                  (void*)&jmin, (void*)&jmax, (void*)&b, (void*)&t, (void*)&flags, (void*)&epoch};
  // cooperative launch: every CTA co-resident (the dataflow waits on other CTAs)
  cudaError_t e = cudaLaunchCooperativeKernel((const void*)coarse_solve_flow_kernel, dim3(g),
                                              dim3(256), args, smem, stream);
  bddc_note_launches(1);
  return e == cudaSuccess ? pc_status() : -(int)e;
}

}  // extern "C"
