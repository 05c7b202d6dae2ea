// Vector kernels of the left-preconditioned GMRES driver (reference
// solver.py:262-315): block Gram-Schmidt dots (CGS2 in place of the
// reference's MGS x2, same Krylov space), multi-vector axpy, norms.
// Reductions are two-pass with a fixed order, so runs are bitwise
// reproducible.
#include <cooperative_groups.h>

#include "common.cuh"
#include "bddc_b200.h"

namespace bddc {

constexpr int kDotThreads = 256;
constexpr int kDotMaxVec = 32;  // vectors per pass; larger m loops

// partial[blk][j] = sum_{t in chunk} V_j[t] * w[t], j in [j0, j0 + mv)
__global__ void __launch_bounds__(kDotThreads) multi_dot_kernel(const double* __restrict__ V,
                                                                long long ldv, long long n, int j0,
                                                                int mv,
                                                                const double* __restrict__ w,
                                                                double* __restrict__ partial,
                                                                int stride) {
  __shared__ double red[kDotThreads / 32][kDotMaxVec];
  double acc[kDotMaxVec];
#pragma unroll
  for (int j = 0; j < kDotMaxVec; ++j) acc[j] = 0.0;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (long long)gridDim.x * blockDim.x) {
    const double wt = w[t];
#pragma unroll
    for (int j = 0; j < kDotMaxVec; ++j)
      if (j < mv) acc[j] += V[(long long)(j0 + j) * ldv + t] * wt;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int j = 0; j < kDotMaxVec; ++j) {
    double v = acc[j];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp][j] = v;
  }
  __syncthreads();
  if (threadIdx.x < mv) {
    double s = 0.0;
    for (int k = 0; k < kDotThreads / 32; ++k) s += red[k][threadIdx.x];
    partial[(long long)blockIdx.x * stride + j0 + threadIdx.x] = s;
  }
}

__global__ void reduce_partials_kernel(const double* __restrict__ partial, int nblocks, int m,
                                       int stride, double* __restrict__ out, int accumulate) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  double s = 0.0;
  for (int b = 0; b < nblocks; ++b) s += partial[(long long)b * stride + j];
  out[j] = accumulate ? out[j] + s : s;
}

// w[t] += alpha * sum_j coef[j] * V_j[t]
__global__ void multi_axpy_kernel(const double* __restrict__ V, long long n, int m,
                                  const double* __restrict__ coef, double alpha,
                                  double* __restrict__ w) {
  extern __shared__ double cf[];
  for (int j = threadIdx.x; j < m; j += blockDim.x) cf[j] = coef[j];
  __syncthreads();
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (long long)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < m; ++j) s += cf[j] * V[(long long)j * n + t];
    w[t] += alpha * s;
  }
}

// out[t] = a[t] * s  with s = scale_num / scale_den[0]   (device scalar)
__global__ void scale_copy_kernel(const double* __restrict__ a, long long n,
                                  const double* __restrict__ den, double* __restrict__ out) {
  const double s = 1.0 / den[0];
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (long long)gridDim.x * blockDim.x)
    out[t] = a[t] * s;
}

__global__ void sqrt_kernel(double* x) { x[0] = sqrt(x[0]); }

__global__ void sqrt_n_kernel(double* x, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = sqrt(x[i]);
}

// halo / slot-exchange packing: dst[i] = src[idx[i]]
__global__ void gather_idx_kernel(const double* __restrict__ src, const long long* __restrict__ idx,
                                  long long n, double* __restrict__ dst) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] = src[idx[i]];
}

// unpacking: dst[idx[i]] = src[i] (add = 0) or += src[i] (add = 1); idx has no
// duplicates within one call, so the result does not depend on thread order
__global__ void scatter_idx_kernel(double* __restrict__ dst, const long long* __restrict__ idx,
                                   long long n, const double* __restrict__ src, int add) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const long long j = idx[i];
    dst[j] = add ? dst[j] + src[i] : src[i];
  }
}

// One GMRES step of the Hessenberg least-squares problem by Givens rotations
// (replaces the per-step host lstsq/gelsd of solver.py:297 with the
// mathematically identical QR recurrence; one CTA).  Column m-1 of H is
// h = h1[0:m] + h2[0:m] (the two classical Gram-Schmidt passes) with
// subdiagonal hn = h2[m].  R: column-major, ldr rows (upper triangular);
// cs/sn: rotations; g: rotated beta e1 (g[0] = beta set by the caller);
// y = R^-1 g[0:m]; out[0] = |g[m]| (the least-squares residual), out[1] = hn.
__global__ void gmres_givens_kernel(const double* __restrict__ h1, const double* __restrict__ h2,
                                    int m, int ldr, double* __restrict__ R, double* __restrict__ cs,
                                    double* __restrict__ sn, double* __restrict__ g,
                                    double* __restrict__ y, double* __restrict__ out) {
  __shared__ double col[1024];
  __shared__ double ys[1024];
  double* Rc = R + (long long)(m - 1) * ldr;
  if (threadIdx.x == 0) {
    for (int i = 0; i < m; ++i) col[i] = h1[i] + h2[i];
    const double hn = h2[m];
    for (int i = 0; i + 1 < m; ++i) {
      const double a = col[i], b = col[i + 1];
      col[i] = cs[i] * a + sn[i] * b;
      col[i + 1] = -sn[i] * a + cs[i] * b;
    }
    const double a = col[m - 1];
    const double r = hypot(a, hn);
    const double c = r > 0.0 ? a / r : 1.0, s = r > 0.0 ? hn / r : 0.0;
    cs[m - 1] = c;
    sn[m - 1] = s;
    col[m - 1] = r;
    const double gm = g[m - 1];
    g[m - 1] = c * gm;
    g[m] = -s * gm;
    for (int i = 0; i < m; ++i) Rc[i] = col[i];
    out[0] = fabs(g[m]);
    out[1] = hn;
  }
  __syncthreads();
  // back substitution, one warp: y_i = (g_i - sum_{k>i} R[i,k] y_k) / R[i,i]
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    for (int i = m - 1; i >= 0; --i) {
      double acc = 0.0;
      for (int k = i + 1 + lane; k < m; k += 32) acc += R[(long long)k * ldr + i] * ys[k];
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) ys[i] = (g[i] - acc) / R[(long long)i * ldr + i];
      __syncwarp();
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < m; i += blockDim.x) y[i] = ys[i];
}

// Givens step of the Hessenberg least-squares recurrence (see
// gmres_givens_kernel), run by one CTA; col / ys: m doubles of shared memory.
BDDC_DEV void givens_step(const double* h1, const double* h2, int m, int ldr, double* R, double* cs,
                          double* sn, double* g, double* y, double* out, double* col, double* ys) {
  double* Rc = R + (long long)(m - 1) * ldr;
  if (threadIdx.x == 0) {
    for (int i = 0; i < m; ++i) col[i] = h1[i] + h2[i];
    const double hn = h2[m];
    for (int i = 0; i + 1 < m; ++i) {
      const double a = col[i], b = col[i + 1];
      col[i] = cs[i] * a + sn[i] * b;
      col[i + 1] = -sn[i] * a + cs[i] * b;
    }
    const double a = col[m - 1];
    const double r = hypot(a, hn);
    const double c = r > 0.0 ? a / r : 1.0, s = r > 0.0 ? hn / r : 0.0;
    cs[m - 1] = c;
    sn[m - 1] = s;
    col[m - 1] = r;
    const double gm = g[m - 1];
    g[m - 1] = c * gm;
    g[m] = -s * gm;
    for (int i = 0; i < m; ++i) Rc[i] = col[i];
    out[0] = fabs(g[m]);
    out[1] = hn;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    for (int i = m - 1; i >= 0; --i) {
      double acc = 0.0;
      for (int k = i + 1 + lane; k < m; k += 32) acc += R[(long long)k * ldr + i] * ys[k];
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) ys[i] = (g[i] - acc) / R[(long long)i * ldr + i];
      __syncwarp();
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < m; i += blockDim.x) y[i] = ys[i];
}

// One GMRES step after w = M^-1 S_hat v_(m-1), in ONE cooperative launch
// (grid-wide barriers instead of ~17 kernel boundaries):
//   h1 = V^T w; w -= V h1; h2 = V^T w; w -= V h2; hn = ||w||   (CGS2)
//   Givens update of the least-squares recurrence, y            (CTA 0)
//   V_m = w / hn;  tres = ||rhs - U y||   (U = S_hat V: the true residual)
// CTA b owns the entries [b * chunk, (b + 1) * chunk) of every vector and keeps
// its piece of w in shared memory.  Reductions: per-CTA partials in a fixed
// order, then every CTA sums the partials of all CTAs in the same fixed order
// (bitwise reproducible, identical in every CTA).
constexpr int kStepThreads = 256;

BDDC_DEV void step_dots(const double* __restrict__ Vb, long long ldv, long long t0, int len, int m,
                        const double* wsm, double* red, double* part) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int j = 0; j < m; ++j) {
    const double* v = Vb + (long long)j * ldv + t0;
    double s = 0.0;
    for (int i = threadIdx.x; i < len; i += kStepThreads) s = fma(v[i], wsm[i], s);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) red[warp * m + j] = s;
  }
  __syncthreads();
  for (int j = threadIdx.x; j < m; j += kStepThreads) {
    double s = 0.0;
    for (int k = 0; k < kStepThreads / 32; ++k) s += red[k * m + j];
    part[(long long)blockIdx.x * m + j] = s;
  }
  __syncthreads();
}

// dst[j] = sum_b part[b * cnt + j], b in a fixed order (lane-strided, then a tree)
BDDC_DEV void step_reduce(const double* part, int nblk, int cnt, double* dst) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int j = warp; j < cnt; j += kStepThreads / 32) {
    double s = 0.0;
    for (int b = lane; b < nblk; b += 32) s += __ldcg(part + (long long)b * cnt + j);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) dst[j] = s;
  }
  __syncthreads();
}

BDDC_DEV void step_axpy(const double* __restrict__ Vb, long long ldv, long long t0, int len, int m,
                        const double* coef, double* wsm) {
  for (int i = threadIdx.x; i < len; i += kStepThreads) {
    double s = 0.0;
    for (int j = 0; j < m; ++j) s = fma(coef[j], Vb[(long long)j * ldv + t0 + i], s);
    wsm[i] -= s;
  }
  __syncthreads();
}

BDDC_DEV double step_block_sum(double s, double* red) {
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  double t = 0.0;
  for (int k = 0; k < kStepThreads / 32; ++k) t += red[k];
  __syncthreads();
  return t;
}

__global__ void __launch_bounds__(kStepThreads) gmres_step_kernel(
    const double* __restrict__ V, const double* __restrict__ U, long long ldv, long long n, int m,
    int chunk, const double* __restrict__ w, const double* __restrict__ rhs, double* h1, double* h2,
    int ldr, double* R, double* cs, double* sn, double* g, double* y, double* out, double* tres,
    double* vnext, double* partial) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double ssm[];
  double* wsm = ssm;                       // chunk
  double* hs = wsm + chunk;                // m + 1
  double* red = hs + m + 1;                // 8 * m (>= 8)
  const int nblk = gridDim.x;
  const long long t0 = (long long)blockIdx.x * chunk;
  const int len = (int)max(0ll, min((long long)chunk, n - t0));
  double* pA = partial;
  double* pB = pA + (long long)nblk * m;
  double* pC = pB + (long long)nblk * m;
  double* pD = pC + nblk;
  for (int i = threadIdx.x; i < len; i += kStepThreads) wsm[i] = w[t0 + i];
  __syncthreads();
  step_dots(V, ldv, t0, len, m, wsm, red, pA);
  grid.sync();
  step_reduce(pA, nblk, m, hs);
  if (blockIdx.x == 0)
    for (int j = threadIdx.x; j < m; j += kStepThreads) h1[j] = hs[j];
  step_axpy(V, ldv, t0, len, m, hs, wsm);
  step_dots(V, ldv, t0, len, m, wsm, red, pB);
  grid.sync();
  step_reduce(pB, nblk, m, hs);
  if (blockIdx.x == 0)
    for (int j = threadIdx.x; j < m; j += kStepThreads) h2[j] = hs[j];
  step_axpy(V, ldv, t0, len, m, hs, wsm);
  {
    double s = 0.0;
    for (int i = threadIdx.x; i < len; i += kStepThreads) s = fma(wsm[i], wsm[i], s);
    s = step_block_sum(s, red);
    if (threadIdx.x == 0) pC[blockIdx.x] = s;
  }
  grid.sync();
  step_reduce(pC, nblk, 1, hs + m);
  const double hn = sqrt(hs[m]);
  if (blockIdx.x == 0) {
    if (threadIdx.x == 0) h2[m] = hn;
    __syncthreads();
    givens_step(h1, h2, m, ldr, R, cs, sn, g, y, out, red, red + m);
  }
  {
    const double inv = 1.0 / hn;
    for (int i = threadIdx.x; i < len; i += kStepThreads) vnext[t0 + i] = wsm[i] * inv;
  }
  grid.sync();
  for (int j = threadIdx.x; j < m; j += kStepThreads) hs[j] = __ldcg(y + j);
  __syncthreads();
  {
    double s = 0.0;
    for (int i = threadIdx.x; i < len; i += kStepThreads) {
      double rv = rhs[t0 + i];
      for (int j = 0; j < m; ++j) rv = fma(-hs[j], U[(long long)j * ldv + t0 + i], rv);
      s = fma(rv, rv, s);
    }
    s = step_block_sum(s, red);
    if (threadIdx.x == 0) pD[blockIdx.x] = s;
  }
  grid.sync();
  if (blockIdx.x == 0) {
    step_reduce(pD, nblk, 1, hs);
    if (threadIdx.x == 0) tres[0] = sqrt(hs[0]);
  }
}

}  // namespace bddc

using namespace bddc;

static int kr_status() {
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : -(int)e;
}

extern "C" {

// h[0:m] (+)= V[:, 0:m]^T w over the first n entries of each row of V
// (row stride ldv).  partial: nblocks * m doubles workspace.
int bddc_multi_dot_ld(const double* V, long long ldv, long long n, int m, const double* w,
                      double* h, double* partial, int nblocks, int accumulate,
                      cudaStream_t stream) {
  if (m <= 0) return 0;
  for (int j0 = 0; j0 < m; j0 += kDotMaxVec) {
    const int mv = min(kDotMaxVec, m - j0);
    multi_dot_kernel<<<nblocks, kDotThreads, 0, stream>>>(V, ldv, n, j0, mv, w, partial, m); bddc_note_launches(1);
  }
  reduce_partials_kernel<<<ceil_div(m, 128), 128, 0, stream>>>(partial, nblocks, m, m, h, accumulate); bddc_note_launches(1);
  return kr_status();
}

int bddc_multi_dot(const double* V, long long n, int m, const double* w, double* h,
                   double* partial, int nblocks, int accumulate, cudaStream_t stream) {
  return bddc_multi_dot_ld(V, n, n, m, w, h, partial, nblocks, accumulate, stream);
}

int bddc_multi_axpy(const double* V, long long n, int m, const double* coef, double alpha,
                    double* w, cudaStream_t stream) {
  if (m <= 0 || n <= 0) return 0;
  const int blocks = min(ceil_div(n, 256), 148 * 8);
  multi_axpy_kernel<<<blocks, 256, m * sizeof(double), stream>>>(V, n, m, coef, alpha, w); bddc_note_launches(1);
  return kr_status();
}

int bddc_norm2(const double* w, long long n, double* out, double* partial, int nblocks,
               cudaStream_t stream) {
  int st = bddc_multi_dot(w, n, 1, w, out, partial, nblocks, 0, stream);
  if (st) return st;
  sqrt_kernel<<<1, 1, 0, stream>>>(out); bddc_note_launches(1);
  return kr_status();
}

int bddc_gmres_givens(const double* h1, const double* h2, int m, int ldr, double* R, double* cs,
                      double* sn, double* g, double* y, double* out, cudaStream_t stream) {
  if (m <= 0 || m > 1023) return -(int)cudaErrorInvalidValue;
  gmres_givens_kernel<<<1, 128, 0, stream>>>(h1, h2, m, ldr, R, cs, sn, g, y, out);
  bddc_note_launches(1);
  return kr_status();
}

int bddc_gmres_step_blocks(void) {
  static PerDeviceInt cached;
  return cached.get([] {
    int dev = current_device(), sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms > 0 ? 2 * sms : 1;
  });
}

int bddc_gmres_step(const double* V, const double* U, long long ldv, long long n, int m,
                    const double* w, const double* rhs, double* h1, double* h2, int ldr, double* R,
                    double* cs, double* sn, double* g, double* y, double* out, double* tres,
                    double* vnext, double* partial, cudaStream_t stream) {
  if (m <= 0 || m > 1023 || n <= 0) return -(int)cudaErrorInvalidValue;
  int nblk = bddc_gmres_step_blocks();
  int chunk = (int)((n + nblk - 1) / nblk);
  chunk = (chunk + 1) & ~1;
  const size_t smem = ((size_t)chunk + 10 * (size_t)m + 16) * sizeof(double);
  if (smem > 200 * 1024) return 1;  // vectors too long for the resident chunks: caller uses the unfused kernels
  static PerDeviceOnce once;
  once([&] {
    cudaFuncSetAttribute(gmres_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  });
  int per_sm = 0, sms = nblk / 2;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gmres_step_kernel, kStepThreads, smem);
  if (per_sm < 2) return 1;
  (void)sms;
  void* args[] = {(void*)&V,   (void*)&U,  (void*)&ldv, (void*)&n,    (void*)&m,   (void*)&chunk,
                  (void*)&w,   (void*)&rhs, (void*)&h1, (void*)&h2,   (void*)&ldr, (void*)&R,
                  (void*)&cs,  (void*)&sn, (void*)&g,   (void*)&y,    (void*)&out, (void*)&tres,
                  (void*)&vnext, (void*)&partial};
  cudaError_t e = cudaLaunchCooperativeKernel((const void*)gmres_step_kernel, dim3(nblk),
                                              dim3(kStepThreads), args, smem, stream);
  bddc_note_launches(1);
  return e == cudaSuccess ? 0 : -(int)e;
}

int bddc_sqrt_inplace(double* x, int n, cudaStream_t stream) {
  if (n <= 0) return 0;
  sqrt_n_kernel<<<ceil_div(n, 128), 128, 0, stream>>>(x, n); bddc_note_launches(1);
  return kr_status();
}

int bddc_gather_idx(const double* src, const long long* idx, long long n, double* dst,
                    cudaStream_t stream) {
  if (n <= 0) return 0;
  gather_idx_kernel<<<min(ceil_div(n, 256), 148 * 8), 256, 0, stream>>>(src, idx, n, dst);
  bddc_note_launches(1);
  return kr_status();
}

int bddc_scatter_idx(double* dst, const long long* idx, long long n, const double* src, int add,
                     cudaStream_t stream) {
  if (n <= 0) return 0;
  scatter_idx_kernel<<<min(ceil_div(n, 256), 148 * 8), 256, 0, stream>>>(dst, idx, n, src, add);
  bddc_note_launches(1);
  return kr_status();
}

int bddc_scale_copy(const double* a, long long n, const double* den, double* out,
                    cudaStream_t stream) {
  if (n <= 0) return 0;
  scale_copy_kernel<<<min(ceil_div(n, 256), 148 * 8), 256, 0, stream>>>(a, n, den, out); bddc_note_launches(1);
  return kr_status();
}

}  // extern "C"
