// SUPG-stabilised P1 element blocks on the device (the
// assembly that feeds the hot path).  Restates reference
// pkg/src/adbddc/discretization.py:91-158 (p1_gradients, stabilization,
// element_contributions) for coefficient fields the device can evaluate:
// affine velocity a(x) = A x + a0, constant reaction c and source f, and a
// viscosity per element (nu[e] = nu_tab[e % nu_period]).
//
// One thread per element: 4 vertices -> gradients and volume (adjugate
// inverse of the edge matrix), 4-point degree-2 quadrature, Peclet-switched
// least-squares weight, 4x4 block and 4-vector.  Writes Ke (m x 16) and
// Fe (m x 4) -- the inputs of bddc_local_assemble -- so the per-step upload
// is the mesh and the coefficient data instead of 20 doubles per element.
#include "common.cuh"
#include "bddc_b200.h"

namespace bddc {

struct SupgFields {
  double A[9];   // velocity matrix (row-major)
  double a0[3];  // velocity offset
  double c, f;   // reaction, source
  double cdiv;   // c - div(a)/2 if the caller gives div(a), else c
  double tau;
};

__global__ void __launch_bounds__(128) supg_elements_kernel(
    const double* __restrict__ nodes, const long long* __restrict__ conn, long long m,
    const double* __restrict__ nu_tab, long long nu_period, SupgFields cf, double* __restrict__ Ke,
    double* __restrict__ Fe, unsigned long long* __restrict__ bad) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m) return;
  constexpr double QA = 0.5854101966249685, QB = 0.13819660112501053;
  double v[4][3];
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const long long nd = conn[e * 4 + a];
#pragma unroll
    for (int d = 0; d < 3; ++d) v[a][d] = nodes[nd * 3 + d];
  }
  // E rows = v_k - v_0 (k = 1..3); G[k] = column k-1 of E^-1; G[0] = -sum
  double E[3][3];
#pragma unroll
  for (int k = 0; k < 3; ++k)
#pragma unroll
    for (int d = 0; d < 3; ++d) E[k][d] = v[k + 1][d] - v[0][d];
  const double c00 = E[1][1] * E[2][2] - E[1][2] * E[2][1];
  const double c01 = E[1][2] * E[2][0] - E[1][0] * E[2][2];
  const double c02 = E[1][0] * E[2][1] - E[1][1] * E[2][0];
  const double det = E[0][0] * c00 + E[0][1] * c01 + E[0][2] * c02;
  const double vol = det / 6.0;
  if (!(vol > 0.0)) {
    atomicMin(bad, (unsigned long long)e);
    return;
  }
  const double id = 1.0 / det;
  // inverse = adj(E) / det; Einv[d][k] = cof[k][d] / det
  double inv[3][3];
  inv[0][0] = c00 * id;
  inv[1][0] = c01 * id;
  inv[2][0] = c02 * id;
  inv[0][1] = (E[0][2] * E[2][1] - E[0][1] * E[2][2]) * id;
  inv[1][1] = (E[0][0] * E[2][2] - E[0][2] * E[2][0]) * id;
  inv[2][1] = (E[0][1] * E[2][0] - E[0][0] * E[2][1]) * id;
  inv[0][2] = (E[0][1] * E[1][2] - E[0][2] * E[1][1]) * id;
  inv[1][2] = (E[0][2] * E[1][0] - E[0][0] * E[1][2]) * id;
  inv[2][2] = (E[0][0] * E[1][1] - E[0][1] * E[1][0]) * id;
  double G[4][3];
#pragma unroll
  for (int k = 1; k < 4; ++k)
#pragma unroll
    for (int d = 0; d < 3; ++d) G[k][d] = inv[d][k - 1];  // grad lambda_k = column k of E^-1
#pragma unroll
  for (int d = 0; d < 3; ++d) G[0][d] = -(G[1][d] + G[2][d] + G[3][d]);
  const double nu = nu_tab[e % nu_period];
  // element diameter and the velocity bound over vertices + centroid
  double h = 0.0;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = a + 1; b < 4; ++b) {
      double s = 0.0;
#pragma unroll
      for (int d = 0; d < 3; ++d) s += (v[a][d] - v[b][d]) * (v[a][d] - v[b][d]);
      h = fmax(h, sqrt(s));
    }
  double anorm = 0.0;
#pragma unroll
  for (int s = 0; s < 5; ++s) {
    double p[3];
#pragma unroll
    for (int d = 0; d < 3; ++d)
      p[d] = s < 4 ? v[s][d] : 0.25 * (v[0][d] + v[1][d] + v[2][d] + v[3][d]);
    double n2 = 0.0;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const double ai = cf.A[3 * i] * p[0] + cf.A[3 * i + 1] * p[1] + cf.A[3 * i + 2] * p[2] + cf.a0[i];
      n2 += ai * ai;
    }
    anorm = fmax(anorm, sqrt(n2));
  }
  const bool advective = h * anorm / (2.0 * nu) >= 1.0;
  const double C = advective ? cf.tau * h / (2.0 * anorm) : cf.tau * h * h / (4.0 * nu);
  // quadrature: points q_i = sum_j Q[i][j] v_j (Q = QA on the diagonal, QB off it)
  const double w = vol / 4.0;
  double adv[4][4], Lq[4][4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    double p[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < 4; ++j) s += (j == q ? QA : QB) * v[j][d];
      p[d] = s;
    }
    double a[3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
      a[i] = cf.A[3 * i] * p[0] + cf.A[3 * i + 1] * p[1] + cf.A[3 * i + 2] * p[2] + cf.a0[i];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      adv[q][j] = a[0] * G[j][0] + a[1] * G[j][1] + a[2] * G[j][2];
      Lq[q][j] = adv[q][j] + cf.c * (j == q ? QA : QB);
    }
  }
  double* K = Ke + e * 16;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const double gg = G[i][0] * G[j][0] + G[i][1] * G[j][1] + G[i][2] * G[j][2];
      double mass = 0.0, tij = 0.0, tji = 0.0, ls = 0.0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double qi = q == i ? QA : QB, qj = q == j ? QA : QB;
        mass += w * cf.cdiv * qi * qj;
        tij += w * qi * adv[q][j];
        tji += w * qj * adv[q][i];
        ls += w * Lq[q][i] * Lq[q][j];
      }
      K[i * 4 + j] = gg * (nu * vol) + mass + 0.5 * (tij - tji) + C * ls;
    }
    double fi = 0.0, fs = 0.0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double wf = w * cf.f;
      fi += wf * (q == i ? QA : QB);
      fs += wf * Lq[q][i];
    }
    Fe[e * 4 + i] = fi + C * fs;
  }
}

}  // namespace bddc

using namespace bddc;

extern "C" int bddc_supg_elements(const double* nodes, const long long* conn, long long m,
                                  const double* nu_tab, long long nu_period, const double* fields,
                                  double* Ke, double* Fe, unsigned long long* bad_element,
                                  cudaStream_t stream) {
  if (m <= 0) return 0;
  SupgFields cf;
  for (int i = 0; i < 9; ++i) cf.A[i] = fields[i];
  for (int i = 0; i < 3; ++i) cf.a0[i] = fields[9 + i];
  cf.c = fields[12];
  cf.f = fields[13];
  cf.cdiv = fields[14];
  cf.tau = fields[15];
  supg_elements_kernel<<<(unsigned)((m + 127) / 128), 128, 0, stream>>>(nodes, conn, m, nu_tab,
                                                                        nu_period, cf, Ke, Fe,
                                                                        bad_element);
  bddc_note_launches(1);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : -(int)e;
}
