// Coarse solve through block-inverse operators (the latency-bound Amdahl term
// of the preconditioner apply, reference lu_solve(coarse_lu) solver.py:192).
//
// bddc_coarse_factor leaves C = L diag(P^-1) U in 64-wide panels: L block unit
// lower (panel columns L' = A21 P_k), U block unit upper (pivot rows
// W = P_k A12), P_k the inverse pivot blocks.  Rows are grouped into blocks of
// kCB = 1024 rows (16 panels).  For block D (rows [D*kCB, D*kCB + h)):
//
//   F_D = Linv_DD [ L_(D, cl_D : D*kCB) | I_h ]        h x (wF + h)
//   G_D = Uinv_DD [ P_D | W_(D, D*kCB + h : cu_D) ]    h x (cu_D - D*kCB)
//
// (Linv_DD / Uinv_DD: inverses of the unit block-triangular diagonal blocks,
// P_D = blockdiag of the panel P_k).  Then
//   forward   z_D = F_D[:, wF:] b_D - F_D[:, :wF] z[cl_D : D*kCB]
//   backward  x_D = G_D[:, :h] z_D - G_D[:, h:]  x[D*kCB + h : cu_D]
// so each block of 512 unknowns is ONE row-parallel GEMV that depends on the
// previous block only through its kCB newest values: 2 * ceil(n / kCB)
// dependent steps instead of 2 * ceil(n / 64) dependent triangular panels.
// F and G are built once per preconditioner with the DMMA tile GEMM (the
// diagonal blocks have identity 64 x 64 diagonal blocks, so the block
// triangular solves are pure GEMM sequences).
#include <cooperative_groups.h>

#include "common.cuh"
#include "bddc_b200.h"
#include "tile_mma.cuh"
#include "reg_gj.cuh"

namespace bddc {

// ---------------------------------------------------------------------------
// Envelope LU (no pivoting) in 64-wide panels with a one-panel lookahead.
// Per panel k: [W = P_k A12 row tiles + L' = A21 P_(k-1) of the previous
// panel] in one launch, then [A22 -= A21 W, with CTA 0 updating the next
// diagonal block first and inverting it: P_(k+1)] in a second launch, so the
// pivot inverse and the column scaling leave the critical path.
// ---------------------------------------------------------------------------
#ifndef BDDC_COARSE_PDL
#define BDDC_COARSE_PDL 1  // programmatic dependent launch of the panel kernels
#endif

// Panel kernels may be launched before their predecessor finishes
// (programmatic stream serialisation): wait for it before touching memory.
BDDC_DEV void wait_prev_grid() {
#if BDDC_COARSE_PDL
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
#endif
}

union CoarseFactorSmem {
  TileSmem tile;
  MmaGjSmem gj;
};

BDDC_DEV void coarse_pivot(double* M, int n, int k, double* pinv, double* piv_out, int* status,
                           CoarseFactorSmem& sm) {
  const int w = min(kTile, n - k);
  const bool bad = reg_gj64(M + (long long)k * n + k, n, w, pinv + (long long)(k / kTile) * kTile * kTile,
                            kTile, 0, piv_out + k, sm.gj);
  if (threadIdx.x == 0 && bad && status) atomicCAS(status, 0, (int)kSingularPivot);
}

__global__ void __launch_bounds__(kTileThreads) coarse_pivot_kernel(double* M, int n, int k,
                                                                    double* pinv, double* piv_out,
                                                                    int* status) {
  extern __shared__ __align__(16) unsigned char cf_raw[];
  wait_prev_grid();
  coarse_pivot(M, n, k, pinv, piv_out, status, *reinterpret_cast<CoarseFactorSmem*>(cf_raw));
}

// blocks [0, trow): W row tiles of panel k (cols [k + w, lim));
// blocks [trow, ...): L' = A21 P_kp on rows [kp + 64, limp) of panel kp = k - 64
__global__ void __launch_bounds__(kTileThreads, kTileMinBlocks) coarse_row_scale_kernel(
    double* M, int n, int k, int lim, int trow, int limp, const double* pinv) {
  extern __shared__ __align__(16) unsigned char cf_raw[];
  TileSmem& sm = reinterpret_cast<CoarseFactorSmem*>(cf_raw)->tile;
  wait_prev_grid();
  const int w = min(kTile, n - k);
  if ((int)blockIdx.x < trow) {
    const int c0 = k + w + blockIdx.x * kTile;
    if (c0 >= lim) return;
    double* C = M + (long long)k * n + c0;
    tile_mma(C, n, w, min(kTile, lim - c0), pinv + (long long)(k / kTile) * kTile * kTile, kTile, C,
             n, w, 1.0, 0.0, sm);
  } else {
    const int kp = k - kTile;
    const int r0 = k + (blockIdx.x - trow) * kTile;
    if (kp < 0 || r0 >= limp) return;
    double* C = M + (long long)r0 * n + kp;
    tile_mma(C, n, min(kTile, limp - r0), kTile, C, n, pinv + (long long)(kp / kTile) * kTile * kTile,
             kTile, kTile, 1.0, 0.0, sm);
  }
}

// A22 -= A21 W over [k + w, lim)^2; CTA 0 owns the next diagonal block and
// inverts it right after its update (next != 0)
__global__ void __launch_bounds__(kTileThreads, kTileMinBlocks) coarse_trail_pivot_kernel(
    double* M, int n, int k, int lim, int next, double* pinv, double* piv_out, int* status) {
  extern __shared__ __align__(16) unsigned char cf_raw[];
  CoarseFactorSmem& sm = *reinterpret_cast<CoarseFactorSmem*>(cf_raw);
  wait_prev_grid();
  const int w = min(kTile, n - k);
  const int s = k + w;
  const int tn_count = (lim - s + kTile - 1) / kTile;
  const int tm = blockIdx.x / tn_count, tn = blockIdx.x - tm * tn_count;
  const int r0 = s + tm * kTile, c0 = s + tn * kTile;
  tile_mma(M + (long long)r0 * n + c0, n, min(kTile, lim - r0), min(kTile, lim - c0),
           M + (long long)r0 * n + k, n, M + (long long)k * n + c0, n, w, -1.0, 1.0, sm.tile);
  if (blockIdx.x == 0 && next) {
    __syncthreads();  // the updated diagonal block is in memory; smem reused
    coarse_pivot(M, n, s, pinv, piv_out, status, sm);
  }
}

constexpr int kCB = 1024;           // rows per block (multiple of 64)
constexpr int kCRC = 8;             // rows per CTA per block
constexpr int kCCta = kCB / kCRC;   // CTAs of the solve (128 <= 148 SMs, co-resident)
constexpr int kCThreads = 256;
constexpr int kCPer = kCB / kCThreads;  // critical-block columns per thread

struct CoarseBlk {
  int DB, h, cl, cu, wF, ldF, ldG;
};

BDDC_DEV CoarseBlk coarse_blk(int D, int n, const int* cl, const int* cu) {
  CoarseBlk b;
  b.DB = D * kCB;
  b.h = min(kCB, n - b.DB);
  b.cl = cl[D];
  b.cu = cu[D];
  b.wF = b.DB - b.cl;
  b.ldF = b.wF + ((b.h + 1) & ~1);
  b.ldG = ((b.cu - b.DB) + 1) & ~1;
  return b;
}

// F_D = [L_(D, cl:DB) | I], G_D = [P_D | W_(D, DB+h:cu)]  (8 rows per CTA)
__global__ void coarse_blk_fill_kernel(const double* __restrict__ A, long long ld, int n,
                                       const double* __restrict__ pinv, long long pstride,
                                       const int* __restrict__ cl, const int* __restrict__ cu,
                                       const long long* __restrict__ foff,
                                       const long long* __restrict__ goff, double* __restrict__ F,
                                       double* __restrict__ G) {
  const int D = blockIdx.y;
  const CoarseBlk k = coarse_blk(D, n, cl, cu);
  for (int r = blockIdx.x * 8; r < min(k.h, blockIdx.x * 8 + 8); ++r) {
    const double* arow = A + (long long)(k.DB + r) * ld;
    double* frow = F + foff[D] + (long long)r * k.ldF;
    for (int c = threadIdx.x; c < k.ldF; c += blockDim.x)
      frow[c] = c < k.wF ? arow[k.cl + c] : (c - k.wF == r ? 1.0 : 0.0);
    double* grow = G + goff[D] + (long long)r * k.ldG;
    const double* prow = pinv + (long long)((k.DB >> 6) + (r >> 6)) * pstride + (r & 63) * 64;
    for (int c = threadIdx.x; c < k.ldG; c += blockDim.x) {
      double v = 0.0;
      if (c < k.h) {
        if ((c >> 6) == (r >> 6)) v = prow[c & 63];
      } else if (k.DB + c < k.cu) {
        v = arow[k.DB + c];
      }
      grow[c] = v;
    }
  }
}

// forward block solve, panel p of every block:  X_p -= L_(p, 0:p) X_(0:p)
__global__ void __launch_bounds__(kTileThreads, kTileMinBlocks) coarse_blk_fwd_kernel(
    const double* __restrict__ A, long long ld, int n, const int* __restrict__ cl,
    const int* __restrict__ cu, const long long* __restrict__ foff, double* __restrict__ F, int p) {
  extern __shared__ __align__(16) unsigned char csm_raw[];
  TileSmem& sm = *reinterpret_cast<TileSmem*>(csm_raw);
  const int D = blockIdx.y;
  const CoarseBlk k = coarse_blk(D, n, cl, cu);
  const int c0 = blockIdx.x * 64;
  // columns of the diagonal part at or beyond 64p are zero in X_(0:p): X_p = Y_p there
  if (64 * p >= k.h || c0 >= k.ldF || c0 >= k.wF + 64 * p) return;
  double* X = F + foff[D];
  tile_mma(X + (long long)64 * p * k.ldF + c0, k.ldF, min(64, k.h - 64 * p), min(64, k.ldF - c0),
           A + (long long)(k.DB + 64 * p) * ld + k.DB, ld, X + c0, k.ldF, 64 * p, -1.0, 1.0, sm);
}

// backward block solve, panel p of every block:  X_p -= W_(p, p+1:) X_(p+1:)
__global__ void __launch_bounds__(kTileThreads, kTileMinBlocks) coarse_blk_bwd_kernel(
    const double* __restrict__ A, long long ld, int n, const int* __restrict__ cl,
    const int* __restrict__ cu, const long long* __restrict__ goff, double* __restrict__ G, int p) {
  extern __shared__ __align__(16) unsigned char csm_raw[];
  TileSmem& sm = *reinterpret_cast<TileSmem*>(csm_raw);
  const int D = blockIdx.y;
  const CoarseBlk k = coarse_blk(D, n, cl, cu);
  const int c0 = blockIdx.x * 64;
  const int r1 = 64 * (p + 1);
  // the P_D part of X_(p+1:) is block upper triangular: zero in columns < 64(p+1)
  if (r1 >= k.h || c0 >= k.ldG || c0 + 64 <= r1) return;
  double* X = G + goff[D];
  tile_mma(X + (long long)64 * p * k.ldG + c0, k.ldG, 64, min(64, k.ldG - c0),
           A + (long long)(k.DB + 64 * p) * ld + k.DB + r1, ld, X + (long long)r1 * k.ldG + c0,
           k.ldG, k.h - r1, -1.0, 1.0, sm);
}

BDDC_DEV unsigned cblk_ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// every thread: wait until counter >= target (thread 0 polls)
BDDC_DEV void cblk_wait(const unsigned* c, unsigned target) {
  if (threadIdx.x == 0)
    while (cblk_ld_acquire(c) < target) __nanosleep(20);
  __syncthreads();
}

// Sum the kCRC partial sums over the CTA; thread 0 writes out[r0 + i] and
// signals the block counter (release).
BDDC_DEV void cblk_finish(double (&s)[kCRC], double* red, double* out, int r0, int nrows,
                          unsigned* counter) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int i = 0; i < kCRC; ++i) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s[i] += __shfl_xor_sync(0xffffffffu, s[i], o);
  }
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < kCRC; ++i) red[warp * kCRC + i] = s[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 0; i < nrows; ++i) {
      double v = 0.0;
#pragma unroll
      for (int w = 0; w < kCThreads / 32; ++w) v += red[w * kCRC + i];
      out[r0 + i] = v;
    }
    __threadfence();
    atomicAdd(counter, 1u);
  }
}

// One cooperative launch of kCCta CTAs: CTA c owns rows [c*kCRC, c*kCRC + kCRC)
// of every block.  Per block: the independent part (right-hand side and every
// block already verified complete) is accumulated first, the 512 columns of
// the newest block are prefetched into registers, then the CTA waits for that
// block's counter and finishes with one GEMV slice and a block reduction.
__global__ void __launch_bounds__(kCThreads, 1) coarse_blk_solve_kernel(
    const double* __restrict__ F, const double* __restrict__ G, int n, int nD,
    const int* __restrict__ cl, const int* __restrict__ cu, const long long* __restrict__ foff,
    const long long* __restrict__ goff, const double* __restrict__ b, double* z, double* x,
    unsigned* cnt, unsigned epoch) {
  __shared__ double red[(kCThreads / 32) * kCRC];
  const int c = blockIdx.x, t = threadIdx.x;
  unsigned* fcnt = cnt;
  unsigned* bcnt = cnt + nD;
  const int r0 = c * kCRC;
  int fpre = 0;  // forward blocks [0, fpre) verified complete by this CTA
  // ---- forward ----
  for (int D = 0; D < nD; ++D) {
    const CoarseBlk k = coarse_blk(D, n, cl, cu);
    const int nr = max(0, min(kCRC, k.h - r0));
    const double* Fb = F + foff[D] + (long long)r0 * k.ldF;
    double s[kCRC];
#pragma unroll
    for (int i = 0; i < kCRC; ++i) s[i] = 0.0;
    const int jc = max(k.cl, k.DB - kCB);  // first column of the newest block
    if (nr > 0) {
      // right-hand side (F_D[:, wF:] is lower triangular: columns <= row)
      for (int j = t; j < r0 + nr; j += kCThreads) {
        const double bv = __ldg(b + k.DB + j);
#pragma unroll
        for (int i = 0; i < kCRC; ++i)
          if (i < nr) s[i] += Fb[(long long)i * k.ldF + k.wF + j] * bv;
      }
      // blocks verified earlier: z columns [cl, jc)
      for (int j = t; j < jc - k.cl; j += kCThreads) {
        const double zv = __ldcg(z + k.cl + j);
#pragma unroll
        for (int i = 0; i < kCRC; ++i)
          if (i < nr) s[i] -= Fb[(long long)i * k.ldF + j] * zv;
      }
    }
    // newest block: prefetch its F slice, wait, finish
    double fr[kCRC][kCPer];
    const int wc = k.DB - jc;
#pragma unroll
    for (int q = 0; q < kCPer; ++q) {
      const int j = t + q * kCThreads;
#pragma unroll
      for (int i = 0; i < kCRC; ++i)
        fr[i][q] = (i < nr && j < wc) ? Fb[(long long)i * k.ldF + (jc - k.cl) + j] : 0.0;
    }
    while (fpre < D) {
      cblk_wait(fcnt + fpre, epoch * (unsigned)((min(kCB, n - fpre * kCB) + kCRC - 1) / kCRC));
      ++fpre;
    }
    if (nr > 0) {
#pragma unroll
      for (int q = 0; q < kCPer; ++q) {
        const int j = t + q * kCThreads;
        const double zv = j < wc ? __ldcg(z + jc + j) : 0.0;
#pragma unroll
        for (int i = 0; i < kCRC; ++i) s[i] -= fr[i][q] * zv;
      }
      cblk_finish(s, red, z + k.DB, r0, nr, fcnt + D);
    }
    __syncthreads();  // red reused next block
  }
  // every forward block (z complete) before the backward sweep
  while (fpre < nD) {
    cblk_wait(fcnt + fpre, epoch * (unsigned)((min(kCB, n - fpre * kCB) + kCRC - 1) / kCRC));
    ++fpre;
  }
  // ---- backward ----
  int bpre = nD;  // backward blocks [bpre, nD) verified complete
  for (int D = nD - 1; D >= 0; --D) {
    const CoarseBlk k = coarse_blk(D, n, cl, cu);
    const int nr = max(0, min(kCRC, k.h - r0));
    const double* Gb = G + goff[D] + (long long)r0 * k.ldG;
    double s[kCRC];
#pragma unroll
    for (int i = 0; i < kCRC; ++i) s[i] = 0.0;
    const int x0 = k.DB + k.h;                 // first coupled column
    const int xe = min(k.cu, x0 + kCB);        // end of the newest (next) block's columns
    if (nr > 0) {
      // G_D[:, :h] z_D (block upper: columns >= 64 * (row panel))
      for (int j = (r0 & ~63) + t; j < k.h; j += kCThreads) {
        const double zv = __ldcg(z + k.DB + j);
#pragma unroll
        for (int i = 0; i < kCRC; ++i)
          if (i < nr) s[i] += Gb[(long long)i * k.ldG + j] * zv;
      }
      // blocks verified earlier: x columns [xe, cu)
      for (int j = xe - k.DB + t; j < k.cu - k.DB; j += kCThreads) {
        const double xv = __ldcg(x + k.DB + j);
#pragma unroll
        for (int i = 0; i < kCRC; ++i)
          if (i < nr) s[i] -= Gb[(long long)i * k.ldG + j] * xv;
      }
    }
    double gr[kCRC][kCPer];
    const int wc = xe - x0;
#pragma unroll
    for (int q = 0; q < kCPer; ++q) {
      const int j = t + q * kCThreads;
#pragma unroll
      for (int i = 0; i < kCRC; ++i)
        gr[i][q] = (i < nr && j < wc) ? Gb[(long long)i * k.ldG + k.h + j] : 0.0;
    }
    while (bpre > D + 1) {
      --bpre;
      cblk_wait(bcnt + bpre, epoch * (unsigned)((min(kCB, n - bpre * kCB) + kCRC - 1) / kCRC));
    }
    if (nr > 0) {
#pragma unroll
      for (int q = 0; q < kCPer; ++q) {
        const int j = t + q * kCThreads;
        const double xv = j < wc ? __ldcg(x + x0 + j) : 0.0;
#pragma unroll
        for (int i = 0; i < kCRC; ++i) s[i] -= gr[i][q] * xv;
      }
      cblk_finish(s, red, x + k.DB, r0, nr, bcnt + D);
    }
    __syncthreads();
  }
}

}  // namespace bddc

using namespace bddc;

// launch with programmatic stream serialisation (the kernel waits on its
// predecessor with griddepcontrol.wait), so its launch overlaps the previous
// panel kernel's tail
template <typename... KArgs, typename... Args>
static void launch_pdl(void (*kern)(KArgs...), int grid, int smem, cudaStream_t stream, Args... args) {
#if BDDC_COARSE_PDL
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kTileThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
#else
  kern<<<grid, kTileThreads, smem, stream>>>(static_cast<KArgs>(args)...);
#endif
}

extern "C" {

int bddc_coarse_factor(double* C, const long long* off, const int* ldv, const int* nv, int n,
                       const int* host_lim, double* pinv, double* piv_out, int* status,
                       cudaStream_t stream) {
  (void)ldv;
  (void)nv;
  if (n <= 0) return 0;
  const int smem = (int)sizeof(CoarseFactorSmem);
  static PerDeviceOnce once;
  once([&] {
    cudaFuncSetAttribute(coarse_pivot_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(coarse_row_scale_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(coarse_trail_pivot_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         smem);
  });
  long long off0 = 0;
  cudaMemcpyAsync(&off0, off, sizeof(long long), cudaMemcpyDeviceToHost, stream);
  cudaStreamSynchronize(stream);
  double* M = C + off0;
  int launches = 1;
  coarse_pivot_kernel<<<1, kTileThreads, smem, stream>>>(M, n, 0, pinv, piv_out, status);
  int limp = 0;  // envelope end of the previous panel (its L' still to scale)
  for (int k = 0; k < n; k += kTile) {
    const int w = min(kTile, n - k);
    const int lim = min(n, host_lim[k / kTile]);
    const int span = lim - k - w;
    const int trow = span > 0 ? ceil_div(span, kTile) : 0;
    const int tsc = (k > 0 && limp > k) ? ceil_div(limp - k, kTile) : 0;
    if (trow + tsc > 0) {
      launch_pdl(coarse_row_scale_kernel, trow + tsc, smem, stream, M, n, k, lim, trow, limp,
                 (const double*)pinv);
      ++launches;
    }
    const int next = k + w < n;
    if (span > 0) {
      const int t = ceil_div(span, kTile);
      launch_pdl(coarse_trail_pivot_kernel, t * t, smem, stream, M, n, k, lim, next, pinv, piv_out,
                 status);
      ++launches;
    } else if (next) {
      launch_pdl(coarse_pivot_kernel, 1, smem, stream, M, n, k + w, pinv, piv_out, status);
      ++launches;
    }
    limp = span > 0 ? lim : 0;
  }
  // the last panel has no rows below it (k + w == n): nothing left to scale
  bddc_note_launches(launches);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : -(int)e;
}

int bddc_coarse_blockinv(const double* A, long long ld, int n, const double* pinv,
                         long long pinv_step_stride, int nD, const int* cl, const int* cu,
                         const long long* foff, const long long* goff, int max_ldf, int max_ldg,
                         double* F, double* G, cudaStream_t stream) {
  if (n <= 0 || nD <= 0) return 0;
  const int smem = (int)sizeof(TileSmem);
  static PerDeviceOnce once;
  once([&] {
    cudaFuncSetAttribute(coarse_blk_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(coarse_blk_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  });
  coarse_blk_fill_kernel<<<dim3(kCB / 8, nD), 256, 0, stream>>>(A, ld, n, pinv, pinv_step_stride,
                                                                cl, cu, foff, goff, F, G);
  int launches = 1;
  const int panels = kCB / 64;
  // the forward (F) and backward (G) chains are independent sequences of small
  // dependent launches: they run side by side, the backward one on a helper
  // stream (per device and host thread) forked / joined with events
  static thread_local cudaStream_t side[PerDeviceOnce::kMaxDev] = {};
  static thread_local cudaEvent_t ev[PerDeviceOnce::kMaxDev][2] = {};
  const int dev = current_device();
  cudaStream_t s2 = stream;
  if (dev >= 0 && dev < PerDeviceOnce::kMaxDev) {
    if (!side[dev]) {
      cudaStreamCreateWithFlags(&side[dev], cudaStreamNonBlocking);
      cudaEventCreateWithFlags(&ev[dev][0], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&ev[dev][1], cudaEventDisableTiming);
    }
    s2 = side[dev];
    cudaEventRecord(ev[dev][0], stream);
    cudaStreamWaitEvent(s2, ev[dev][0], 0);
  }
  for (int p = panels - 2; p >= 0; --p) {
    coarse_blk_bwd_kernel<<<dim3(ceil_div(max_ldg, 64), nD), kTileThreads, smem, s2>>>(
        A, ld, n, cl, cu, goff, G, p);
    ++launches;
  }
  for (int p = 1; p < panels; ++p) {
    coarse_blk_fwd_kernel<<<dim3(ceil_div(max_ldf, 64), nD), kTileThreads, smem, stream>>>(
        A, ld, n, cl, cu, foff, F, p);
    ++launches;
  }
  if (s2 != stream) {
    cudaEventRecord(ev[dev][1], s2);
    cudaStreamWaitEvent(stream, ev[dev][1], 0);
  }
  bddc_note_launches(launches);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : -(int)e;
}

int bddc_coarse_block_rows(void) { return kCB; }

int bddc_coarse_solve_blockinv(const double* F, const double* G, int n, int nD, const int* cl,
                               const int* cu, const long long* foff, const long long* goff,
                               const double* b, double* z, double* x, int* counters, int epoch,
                               cudaStream_t stream) {
  if (n <= 0 || nD <= 0) return 0;
  unsigned ep = (unsigned)epoch;
  unsigned* cnt = reinterpret_cast<unsigned*>(counters);
  void* args[] = {(void*)&F,    (void*)&G,  (void*)&n,   (void*)&nD,  (void*)&cl,
                  (void*)&cu,   (void*)&foff, (void*)&goff, (void*)&b, (void*)&z,
                  (void*)&x,    (void*)&cnt, (void*)&ep};
  // cooperative launch: all kCCta CTAs co-resident (they wait on each other's counters)
  cudaError_t e = cudaLaunchCooperativeKernel((const void*)coarse_blk_solve_kernel, dim3(kCCta),
                                              dim3(kCThreads), args, 0, stream);
  bddc_note_launches(1);
  return e == cudaSuccess ? 0 : -(int)e;
}

}  // extern "C"
