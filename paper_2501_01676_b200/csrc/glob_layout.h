// Workspace sizes (in doubles) of the per-glob kernels in globs.cu.
// The Python host mirrors these formulas (paper_2501_01676_b200/_layout.py);
// tests/test_layout.py checks both agree through the exported bddc_ws_* calls.
#pragma once

#ifdef __CUDACC__
#define BDDC_HD __host__ __device__ inline
#else
#define BDDC_HD inline
#endif

BDDC_HD long long bddc_rowspace_ws(long long m, long long n) {
  long long mx = m > n ? m : n;
  return 2 * n * n + n + mx + (m <= n ? n * m : m * n + n * n);
}

// old-edge kernel: 7 n^2 + n + max(parallel sum, pencil, row space)
BDDC_HD long long bddc_edge_old_ws(long long n) {
  long long sc = 8 * n * n + 3 * n;
  long long rs = bddc_rowspace_ws(n, n);
  if (rs > sc) sc = rs;
  return 7 * n * n + n + sc + 32 * n + 64;
}

BDDC_HD long long bddc_edge_new_ws(long long ns, long long ne, long long wd, long long nhmax) {
  long long nC = (ns - 1) * ne;
  long long nr = wd - nC;
  long long xd = ne + nhmax;
  long long base = ns * ne * nC + nC * nC + wd * wd + xd * xd + 2 * wd * wd;
  long long sc = 8 * nC * nC + 3 * nC;
  long long pf = 3 * nr * nr + nr;
  if (pf > sc) sc = pf;
  long long rs = bddc_rowspace_ws(nC * (ns - 1), ne);
  if (rs > sc) sc = rs;
  return base + sc + 32 * nC + 64;
}
