// Shared helpers for the B200 (sm_100a) adaptive-BDDC kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#define BDDC_DEV __device__ __forceinline__

extern "C" void bddc_note_launches(int n);

namespace bddc {

// Status codes written by kernels into caller-owned device int arrays
// (one slot per batch member; 0 = ok).
enum Status : int {
  kOk = 0,
  kNotPositiveDefinite = 1,   // Cholesky / LDL^T pivot <= 0 (reference cho_factor failure)
  kSingularPivot = 2,         // zero or non-finite pivot in an unpivoted elimination
  kNotPSD = 3,                // pencil right-hand side not PSD (linalg.py:151-152)
  kNoConvergence = 4,         // Jacobi sweep limit reached
};

BDDC_DEV void set_status(int* status, int idx, int code) {
  if (status) atomicCAS(status + idx, 0, code);
}

// DMMA m8n8k4 (fp64 tensor-core pipe on sm_100a): D = A*B + C.
// a: A[g][t], b: B[t][g], c0/c1: C[g][2t], C[g][2t+1]   (g = lane/4, t = lane%4)
BDDC_DEV void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <typename T>
BDDC_DEV T ld_nc(const T* p) { return __ldg(p); }

inline int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }

inline int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}

// One-time host-side setup per CUDA device (kernel attributes such as
// cudaFuncAttributeMaxDynamicSharedMemorySize apply per device).  The setup
// functions are idempotent, so concurrent first callers may both run them.
struct PerDeviceOnce {
  static constexpr int kMaxDev = 64;
  std::atomic<int> done[kMaxDev] = {};
  template <class F>
  void operator()(F&& f) {
    const int dev = current_device();
    if (dev < 0 || dev >= kMaxDev) {
      f();
      return;
    }
    if (done[dev].load(std::memory_order_acquire)) return;
    f();
    done[dev].store(1, std::memory_order_release);
  }
};

// Per-device cached integer (e.g. an occupancy-derived grid size); 0 = unset.
struct PerDeviceInt {
  static constexpr int kMaxDev = 64;
  std::atomic<int> v[kMaxDev] = {};
  template <class F>
  int get(F&& f) {
    const int dev = current_device();
    if (dev < 0 || dev >= kMaxDev) return f();
    int x = v[dev].load(std::memory_order_acquire);
    if (x == 0) {
      x = f();
      v[dev].store(x, std::memory_order_release);
    }
    return x;
  }
};

}  // namespace bddc
