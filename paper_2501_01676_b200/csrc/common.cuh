// Shared helpers for the B200 (sm_100a) adaptive-BDDC kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

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

}  // namespace bddc
