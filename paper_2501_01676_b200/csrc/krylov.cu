// Vector kernels of the left-preconditioned GMRES driver (reference
// solver.py:262-315): block Gram-Schmidt dots (CGS2 in place of the
// reference's MGS x2, same Krylov space), multi-vector axpy, norms.
// Reductions are two-pass with a fixed order, so runs are bitwise
// reproducible.
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
