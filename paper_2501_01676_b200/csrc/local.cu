// Per-subdomain dense kernels: local assembly, blocked Schur elimination
// (partial LU without pivoting -> S, g), blocked Gauss-Jordan inversion
// (Bsym^-1, dual blocks), extraction and interior recovery.
//
// Reference call sites replaced (see include/bddc_b200.h for the C-ABI):
//   substructuring.py:98-127   local assembly, lifting, splu(A_II), S and g
//   substructuring.py:64-75    cho_factor/cho_solve(Bsym, I)
//   solver.py:318-326          recover_interior (lu_II.solve)
//
// Layout: batch of row-major matrices in one device buffer; matrix b starts
// at base + off[b] with leading dimension ld[b] (variable sizes, "vbatched").
#include "common.cuh"
#include "bddc_b200.h"
#include "tile_mma.cuh"
#include "reg_gj.cuh"

#include <vector>

namespace bddc {

// ---------------------------------------------------------------------------
// local assembly: element 4x4 blocks -> dense [I | B] x [I | B | f] matrix
//
// Deterministic (no atomics; bitwise reproducible run to run), one CTA per
// subdomain:
//  1. the subdomain's element corners are bucketed by local row with a
//     stable counting sort: warp w histograms a contiguous chunk of corners,
//     an exclusive scan over (row, warp) gives every warp its cursor in every
//     row, and each warp places its chunk in order (__match_any_sync ranks
//     lanes with equal rows), so each row's list is in ascending corner order;
//  2. one warp per row accumulates the row in shared memory in that order
//     (lane t adds corner t's four entries, lanes in turn) and writes all ld
//     entries of the row ([I|B] columns, the load column with the Dirichlet
//     lifting, padding), so K needs no memset.
// ---------------------------------------------------------------------------
constexpr int kAsmWarps = 8;
constexpr int kAsmSlots = 16;  // distinct columns per row in the compact row phase (Kuhn: 15)

BDDC_DEV int block_excl_scan_ints(int* a, int n, int* red) {
  // in-place exclusive scan of a[0..n) by the whole CTA; returns the total.
  // red: kAsmWarps + 1 ints of shared scratch
  const int t = threadIdx.x, nt = blockDim.x;
  const int per = (n + nt - 1) / nt;
  const int i0 = min(n, t * per), i1 = min(n, i0 + per);
  int s = 0;
  for (int i = i0; i < i1; ++i) s += a[i];
  const int lane = t & 31, w = t >> 5;
  int x = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) red[w] = x;
  __syncthreads();
  if (t == 0) {
    int run = 0;
    for (int k = 0; k < (nt >> 5); ++k) {
      const int v = red[k];
      red[k] = run;
      run += v;
    }
    red[nt >> 5] = run;
  }
  __syncthreads();
  int run = red[w] + x - s;
  for (int i = i0; i < i1; ++i) {
    const int v = a[i];
    a[i] = run;
    run += v;
  }
  const int total = red[nt >> 5];
  __syncthreads();
  return total;
}

__global__ void __launch_bounds__(kAsmWarps * 32) assemble_rows_kernel(
    double* __restrict__ base, const long long* __restrict__ off, const int* __restrict__ ld,
    const int* __restrict__ nloc, const long long* __restrict__ elem_start,
    const long long* __restrict__ elem_ids, const int* __restrict__ loc4,
    const long long* __restrict__ conn, const double* __restrict__ Ke,
    const double* __restrict__ Fe, const double* __restrict__ gdir, int* __restrict__ lists,
    long long* __restrict__ keys, int nrowbuf, int* __restrict__ overflow, int region0,
    const int* __restrict__ nint, const int* __restrict__ ndeep) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int b = blockIdx.x;
  const int nL = nloc[b], L = ld[b];
  const long long e0 = elem_start[b], e1 = elem_start[b + 1];
  const long long nc = 4 * (e1 - e0);
  const int stride = nL + 1;
  // [region0: warp histograms (counts, then cursors); reused by the compact row
  //  lists] [rowptr nL + 1] [red kAsmWarps + 1] [row buffers]
  int* hist = reinterpret_cast<int*>(smem_raw);
  int* rowptr = reinterpret_cast<int*>(smem_raw + region0);
  int* red = rowptr + stride;
  double* rowbuf = reinterpret_cast<double*>(
      smem_raw + region0 + ((((size_t)(stride + kAsmWarps + 1)) * 4 + 15) & ~(size_t)15));
  int* lst = lists + 4 * e0;
  const long long* eid = elem_ids + e0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  for (int i = threadIdx.x; i < kAsmWarps * stride; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  const long long chunk = (nc + kAsmWarps - 1) / kAsmWarps;
  const long long c0 = min(nc, (long long)warp * chunk), c1 = min(nc, c0 + chunk);
  int* h = hist + warp * stride;
  long long* kp = keys + 4 * e0;
  // pass 1: (row, global corner id) of every corner into keys, per-warp row counts
#pragma unroll 4
  for (long long j = c0 + lane; j < c1; j += 32) {
    const long long gc = eid[j >> 2] * 4 + (j & 3);
    const int r = loc4[gc];
    kp[j] = r < nL ? ((long long)r << 32) | gc : -1;
    if (r < nL) atomicAdd(h + r, 1);  // integer counts: order-independent
  }
  __syncthreads();
  for (int r = threadIdx.x; r < nL; r += blockDim.x) {
    int s = 0;
#pragma unroll
    for (int w = 0; w < kAsmWarps; ++w) s += hist[w * stride + r];
    rowptr[r] = s;
  }
  __syncthreads();
  const int total = block_excl_scan_ints(rowptr, nL, red);
  if (threadIdx.x == 0) rowptr[nL] = total;
  for (int r = threadIdx.x; r < nL; r += blockDim.x) {
    int run = rowptr[r];
#pragma unroll
    for (int w = 0; w < kAsmWarps; ++w) {
      const int v = hist[w * stride + r];
      hist[w * stride + r] = run;
      run += v;
    }
  }
  __syncthreads();
  // stable placement, 32 corners at a time in order
  for (long long jb = c0; jb < c1; jb += 32) {
    const long long j = jb + lane;
    const long long key = j < c1 ? kp[j] : -1;
    const int r = key < 0 ? -1 : (int)(key >> 32);
    const unsigned m = __match_any_sync(0xffffffffu, r);
    const int rank = __popc(m & ((1u << lane) - 1u));
    int pos = 0;
    if (r >= 0) pos = h[r];
    __syncwarp();
    if (r >= 0 && rank == 0) h[r] = pos + __popc(m);
    __syncwarp();
    if (r >= 0) lst[pos + rank] = (int)(key & 0xffffffffll);  // global corner id
  }
  __syncthreads();
  double* M = base + off[b];
  if (nrowbuf == 0) {
    // compact row phase: lane owns a row, keeps its (column, value) pairs in a
    // short shared-memory list (Kuhn meshes: <= 15 columns per row), then the
    // warp zero-fills its 32 rows with coalesced stores and every lane writes
    // its row's nonzeros.  Same summation order as the row-buffer phase below.
    double* lval = reinterpret_cast<double*>(hist) + (size_t)warp * 32 * kAsmSlots;
    int* lcol = reinterpret_cast<int*>(reinterpret_cast<double*>(hist) + kAsmWarps * 32 * kAsmSlots) +
                (size_t)warp * 32 * kAsmSlots;
    const int nd = ndeep ? ndeep[b] : 0, nIb = nint ? nint[b] : nL;
    double* rbuf = rowbuf + (size_t)warp * (L + 2);
    int ovf = 0;
    for (int rb = warp * 32; rb < nL; rb += kAsmWarps * 32) {
      const int r = rb + lane;
      int cnt = 0;
      double fload = 0.0;
      if (r < nL) {
        const int s1 = rowptr[r + 1];
        int gnext = rowptr[r] < s1 ? lst[rowptr[r]] : 0;
        for (int s = rowptr[r]; s < s1; ++s) {
          const int gc = gnext;
          if (s + 1 < s1) gnext = lst[s + 1];  // next corner's id in flight
          const long long e = gc >> 2;
          const int a = gc & 3;
          double fr = Fe[gc];
          double kv[4];
          int kl[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            kv[c] = Ke[e * 16 + a * 4 + c];
            kl[c] = loc4[e * 4 + c];
          }
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const double v = kv[c];
            const int li = kl[c];
            if (li < nL) {
              int t = 0;
              while (t < cnt && lcol[t * 32 + lane] != li) ++t;
              if (t < cnt) {
                lval[t * 32 + lane] += v;
              } else if (cnt < kAsmSlots) {
                lcol[cnt * 32 + lane] = li;
                lval[cnt * 32 + lane] = v;
                ++cnt;
              } else {
                ovf = 1;
              }
            } else {
              fr -= v * gdir[conn[e * 4 + c]];
            }
          }
          fload += fr;
        }
      }
      // dense rows through the warp's shared-memory row buffer: every row of K
      // is written once, with full-line (16-byte vector) stores.  With the
      // two-phase elimination the blocks nobody reads are not written at all:
      // deep rows x interface columns and interface rows x deep columns (both
      // structurally zero; the panel kernels, the extraction and the recovery
      // skip them).
      const int nrows = min(32, nL - rb);
      double2* rb2 = reinterpret_cast<double2*>(rbuf);
      for (int q = 0; q < nrows; ++q) {
        const int rr = rb + q;
        int z0 = 0, z1 = 0;
        if (nd > 0) {
          if (rr < nd) {
            z0 = nIb;
            z1 = nL;
          } else if (rr >= nIb) {
            z1 = nd;
          }
        }
        for (int c = lane; c < (L >> 1); c += 32) rb2[c] = make_double2(0.0, 0.0);
        __syncwarp();
        const int cq = __shfl_sync(0xffffffffu, cnt, q);
        const double fq = __shfl_sync(0xffffffffu, fload, q);
        if (lane < cq) rbuf[lcol[lane * 32 + q]] = lval[lane * 32 + q];
        if (lane == 0) rbuf[nL] = fq;
        __syncwarp();
        double2* row2 = reinterpret_cast<double2*>(M + (long long)rr * L);
        for (int c = lane; c < (L >> 1); c += 32)
          if (!(2 * c >= z0 && 2 * c + 1 < z1)) row2[c] = rb2[c];
        __syncwarp();
      }
    }
    if (ovf && overflow) atomicExch(overflow, 1);
    return;
  }
  if (warp >= nrowbuf) return;
  double* rb = rowbuf + (size_t)warp * L;
  const int nwr = min(nrowbuf, kAsmWarps);
  for (int r = warp; r < nL; r += nwr) {
    for (int c = lane; c < L; c += 32) rb[c] = 0.0;
    __syncwarp();
    const int s0 = rowptr[r], s1 = rowptr[r + 1];
    for (int sb = s0; sb < s1; sb += 32) {
      const int s = sb + lane;
      int col[4] = {-1, -1, -1, -1};
      double val[4] = {0.0, 0.0, 0.0, 0.0};
      double fr = 0.0;
      if (s < s1) {
        const int gc = lst[s];
        const long long e = gc >> 2;
        const int a = gc & 3;
        fr = Fe[gc];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const double v = Ke[e * 16 + a * 4 + c];
          const int li = loc4[e * 4 + c];
          if (li < nL) {
            col[c] = li;
            val[c] = v;
          } else {
            fr -= v * gdir[conn[e * 4 + c]];
          }
        }
      }
      const int cnt = min(32, s1 - sb);
      for (int t = 0; t < cnt; ++t) {
        if (lane == t) {
#pragma unroll
          for (int c = 0; c < 4; ++c)
            if (col[c] >= 0) rb[col[c]] += val[c];
          rb[nL] += fr;
        }
        __syncwarp();
      }
    }
    double* row = M + (long long)r * L;
    for (int c = lane; c < L; c += 32) row[c] = rb[c];
    __syncwarp();
  }
}

static size_t assemble_region0(int max_nl, int nrowbuf) {
  size_t hist_bytes = (size_t)kAsmWarps * (max_nl + 1) * 4;
  if (nrowbuf == 0) {  // compact phase reuses the histogram region for the row lists
    const size_t lists = (size_t)kAsmWarps * 32 * kAsmSlots * 12;
    hist_bytes = hist_bytes > lists ? hist_bytes : lists;
  }
  return (hist_bytes + 15) & ~(size_t)15;
}

static size_t assemble_smem_bytes(int max_nl, int nrowbuf) {
  const size_t ints = (max_nl + 1) + kAsmWarps + 1;
  const int nbuf = nrowbuf == 0 ? kAsmWarps : nrowbuf;  // the compact phase has one per warp
  return assemble_region0(max_nl, nrowbuf) + ((ints * 4 + 15) & ~(size_t)15) +
         (size_t)nbuf * (max_nl + 4) * 8;
}

// ---------------------------------------------------------------------------
// symbolic plan: element-local dof index of every element corner
//   interior node      -> its interior index (iloc_of_node)
//   interface node     -> nI[s] + block offset of its glob in s + position in glob
//   Dirichlet / absent -> 2^30
// ---------------------------------------------------------------------------
__global__ void plan_loc4_kernel(const long long* __restrict__ conn,
                                 const long long* __restrict__ sub_of, long long n_corners,
                                 int s0, const int* __restrict__ iloc_of_node,
                                 const int* __restrict__ glob_of_node,
                                 const int* __restrict__ pos_in_glob,
                                 const int* __restrict__ sh_start, const int* __restrict__ sh_sub,
                                 const int* __restrict__ sh_boff, const long long* __restrict__ nI,
                                 int* __restrict__ loc4) {
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < n_corners;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long nd = conn[idx];
    const int il = iloc_of_node[nd];
    if (il >= 0) {
      loc4[idx] = il;
      continue;
    }
    int v = 1 << 30;
    const int g = glob_of_node[nd];
    if (g >= 0) {
      const int s = (int)sub_of[idx >> 2];
      for (int k = sh_start[g]; k < sh_start[g + 1]; ++k)
        if (sh_sub[k] == s) v = (int)nI[s - s0] + sh_boff[k] + pos_in_glob[nd];
    }
    loc4[idx] = v;
  }
}

// ---------------------------------------------------------------------------
// pivot block inverse (w x w, w <= 64): register block Gauss-Jordan (reg_gj.cuh)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256, 4) pivot_inverse_kernel(
    const double* __restrict__ base, const long long* __restrict__ off, const int* __restrict__ ld,
    const int* __restrict__ npiv, int k, double* __restrict__ pinv, long long pinv_stride,
    int* __restrict__ status, int require_positive, double* __restrict__ piv_out,
    long long piv_stride, int ldo = kTile, int only_small = 0) {
  __shared__ MmaGjSmem sm;
  const int b = blockIdx.x;
  const int w = min(kTile, npiv[b] - k);
  if (w <= 0) return;
  if (only_small && npiv[b] - k > kTile) return;  // wider pivot blocks: the 128-panel route
  const int L = ld[b];
  const double* M = base + off[b] + (long long)k * L + k;
  const bool bad = reg_gj64(M, L, w, pinv + (long long)b * pinv_stride, ldo, require_positive,
                            piv_out ? piv_out + (long long)b * piv_stride + k : nullptr, sm);
  if (threadIdx.x == 0 && bad && status)
    atomicCAS(status + b, 0, require_positive ? (int)kNotPositiveDefinite : (int)kSingularPivot);
}

// ---------------------------------------------------------------------------
// Schur elimination (LU-style, rows below only):
//   W = A11^-1 A12 stored over A12;   A22 -= A21 W
// ---------------------------------------------------------------------------
// Column hole (two-phase elimination, deep interior pivots): the pivot rows of
// the first phase have no entries in columns [h0, h1) (the interface block), so
// the column tiles of a panel step cover [s, h0) and [h1, nc) only.
struct ColHole {
  const int* h0;  // per matrix, null: no hole
  const int* h1;
};

BDDC_DEV int tile_col_count(int s, int nc, int h0, int h1) {
  if (h0 >= h1) return (nc - s + kTile - 1) / kTile;
  return (max(h0 - s, 0) + kTile - 1) / kTile + (max(nc - h1, 0) + kTile - 1) / kTile;
}

// column tile tn of [s, nc) minus [h0, h1): first column and width; false past the end
BDDC_DEV bool tile_cols(int s, int tn, int nc, int h0, int h1, int& c0, int& n) {
  int c = s + tn * kTile, end = nc;
  if (h0 < h1) {
    const int t0 = (max(h0 - s, 0) + kTile - 1) / kTile;  // tiles before the hole
    if (tn < t0) end = h0;
    else c = h1 + (tn - t0) * kTile;
  }
  if (c >= end) return false;
  c0 = c;
  n = min(kTile, end - c);
  return true;
}

__global__ void __launch_bounds__(kTileThreads, kTileMinBlocks) schur_row_kernel(
    double* __restrict__ base, const long long* __restrict__ off, const int* __restrict__ ld,
    const int* __restrict__ npiv, const int* __restrict__ ncols, int k,
    const double* __restrict__ pinv, long long pinv_stride, int lim, ColHole hole) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  TileSmem& sm = *reinterpret_cast<TileSmem*>(smem_raw);
  const int b = blockIdx.y;
  const int w = min(kTile, npiv[b] - k);
  if (w <= 0) return;
  const int nc = min(ncols[b], lim);
  const int h0 = hole.h0 ? hole.h0[b] : 0, h1 = hole.h0 ? hole.h1[b] : 0;
  int c0, n;
  if (!tile_cols(k + w, blockIdx.x, nc, h0, h1, c0, n)) return;
  const int L = ld[b];
  double* C = base + off[b] + (long long)k * L + c0;
  tile_mma(C, L, w, n, pinv + (long long)b * pinv_stride, kTile, C, L, w, 1.0, 0.0, sm);
}

constexpr int kTrailBM = 64;  // row-tile height of the big (mode 0) trailing updates (128 x 64 tiles, 512 threads: measured slower, 34.8 -> 38.2 ms)

// Trailing update of a panel step.  mode 0: rows/cols from k + w, K = w with
// w = min(nbw, npiv - k) (nbw = 64 or 128).  mode 1 (inside a 128-wide panel,
// K = w1 = min(64, npiv - k)): the strip rows [k + w1, k + w), cols from k + w1,
// and (extra CTAs) the column panel rows >= k + w, cols [k + w1, k + w), so that
// the factors of a 128-wide panel are those of two 64-wide panels ("rows below
// only" form: pivot rows W_k = P_k A12^(k), column panels A21^(k)).
// Lookahead (pnext != null): CTA 0 of each matrix owns the next pivot block
// (rows / cols from s) and inverts it right after its tile update, so the
// next panel needs no separate pivot launch.
struct NextPivot {
  double* pinv;           // P of the next pivot block (+ b * stride), null: no lookahead
  long long stride;
  int* status;
  int require_positive;
  double* piv_out;        // scalar pivots (+ b * piv_stride + next k), may be null
  long long piv_stride;
};

template <int BM>
__global__ void __launch_bounds__(BM * 4, BM == 64 ? kTileMinBlocks : 2) schur_trailing_kernel(
    double* __restrict__ base, const long long* __restrict__ off, const int* __restrict__ ld,
    const int* __restrict__ npiv, const int* __restrict__ nrows, const int* __restrict__ ncols,
    int k, int lim, int nbw, int mode, NextPivot nx, ColHole hole) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  TileSmemT<BM>& sm = *reinterpret_cast<TileSmemT<BM>*>(smem_raw);
  const int b = blockIdx.y;
  const int np = npiv[b] - k;
  if (np <= 0) return;
  int w, s, r_begin, r_end;
  const int nc = min(ncols[b], lim);
  if (mode == 0) {
    w = min(nbw, np);
    s = k + w;
    r_begin = s;
    r_end = min(nrows[b], lim);
  } else {
    const int w1 = min(kTile, np), wt = min(2 * kTile, np);
    if (wt <= w1) return;
    w = w1;
    s = k + w1;
    r_begin = k + w1;
    r_end = k + wt;
  }
  const int h0 = hole.h0 ? hole.h0[b] : 0, h1 = hole.h0 ? hole.h1[b] : 0;
  const int tn_count = tile_col_count(s, nc, h0, h1);
  if (tn_count <= 0) return;
  const int L = ld[b];
  double* M = base + off[b];
  if (mode == 1 && (int)blockIdx.x >= tn_count) {
    // the same K = w1 update on the column panel of the second sub-panel below the
    // 128-wide panel: A21^(k2) = A[., k2] - A[., k1] W1[:, k2 block], so that the
    // K = 128 trailing update below multiplies [A[., k1] | A21^(k2)] by [W1; W2]
    // and the factors stay in the 64-panel "rows below only" form
    const int wt = min(2 * kTile, np);
    const int r0 = k + wt + ((int)blockIdx.x - tn_count) * BM;
    const int rend = min(nrows[b], lim);
    if (r0 >= rend) return;
    tile_mma_t<BM>(M + (long long)r0 * L + s, L, min(BM, rend - r0), wt - w,
                   M + (long long)r0 * L + k, L, M + (long long)k * L + s, L, w, -1.0, 1.0, sm);
    return;
  }
  const int tm = blockIdx.x / tn_count, tn = blockIdx.x - tm * tn_count;
  const int r0 = r_begin + tm * BM;
  int c0, cn;
  if (r0 >= r_end || !tile_cols(s, tn, nc, h0, h1, c0, cn)) return;
  tile_mma_t<BM>(M + (long long)r0 * L + c0, L, min(BM, r_end - r0), cn,
                 M + (long long)r0 * L + k, L, M + (long long)k * L + c0, L, w, -1.0, 1.0, sm);
  if (nx.pinv != nullptr && blockIdx.x == 0) {
    const int wn = min(kTile, npiv[b] - s);
    if (wn > 0) {
      __syncthreads();  // tile written; the pipeline smem is free
      static_assert(sizeof(MmaGjSmem) <= sizeof(TileSmemT<BM>), "smem reuse");
      MmaGjSmem& gsm = *reinterpret_cast<MmaGjSmem*>(smem_raw);
      if (threadIdx.x < 256) {  // the register Gauss-Jordan runs on 256 threads (named barrier)
        const bool bad = reg_gj64(M + (long long)s * L + s, L, wn,
                                  nx.pinv + (long long)b * nx.stride, kTile, nx.require_positive,
                                  nx.piv_out ? nx.piv_out + (long long)b * nx.piv_stride + s : nullptr,
                                  gsm);
        if (threadIdx.x == 0 && bad && nx.status)
          atomicCAS(nx.status + b, 0,
                    nx.require_positive ? (int)kNotPositiveDefinite : (int)kSingularPivot);
      }
    }
  }
}

// L' = A21 P_k in place on the panel column rows [k+w, lim) (coarse envelope
// LU: the forward solve then needs no P_k product)
__global__ void __launch_bounds__(kTileThreads, kTileMinBlocks) panel_scale_kernel(double* __restrict__ M,
                                                                   long long ld, int k, int w,
                                                                   int lim,
                                                                   const double* __restrict__ P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  TileSmem& sm = *reinterpret_cast<TileSmem*>(smem_raw);
  const int r0 = k + w + blockIdx.x * kTile;
  if (r0 >= lim) return;
  double* C = M + (long long)r0 * ld + k;
  tile_mma(C, ld, min(kTile, lim - r0), w, C, ld, P, kTile, w, 1.0, 0.0, sm);
}

// ---------------------------------------------------------------------------
// blocked Gauss-Jordan inversion in place (square n x n, no pivoting)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kTileThreads, kTileMinBlocks) gj_row_kernel(
    double* __restrict__ base, const long long* __restrict__ off, const int* __restrict__ ld,
    const int* __restrict__ n, int k, const double* __restrict__ pinv, long long pinv_stride,
    int symmetric) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  TileSmem& sm = *reinterpret_cast<TileSmem*>(smem_raw);
  const int b = blockIdx.y;
  const int w = min(kTile, n[b] - k);
  if (w <= 0) return;
  const int c0 = blockIdx.x * kTile;
  if (c0 >= n[b]) return;
  const int L = ld[b];
  if (c0 == k) {
    // pivot block <- sym(P): written here in the symmetric variant (the update
    // skips it), so that P may be overwritten by the next pivot during the
    // update; otherwise gj_col writes it
    if (symmetric) {
      const double* P = pinv + (long long)b * pinv_stride;
      double* M = base + off[b];
      for (int idx = threadIdx.x; idx < w * w; idx += blockDim.x) {
        const int r = idx / w, c = idx - r * w;
        M[(long long)(k + r) * L + k + c] = 0.5 * (P[r * kTile + c] + P[c * kTile + r]);
      }
    }
    return;
  }
  double* C = base + off[b] + (long long)k * L + c0;
  tile_mma(C, L, w, min(kTile, n[b] - c0), pinv + (long long)b * pinv_stride, kTile, C, L, w, 1.0,
           0.0, sm);
}

// symmetric != 0 (symmetric input): in-place GJ keeps G_JJ and G_KK symmetric
// and G_JK = -G_KJ^T (K = processed pivots), so only tiles tm >= tn are
// computed and each off-diagonal result is mirrored with that sign.
__global__ void __launch_bounds__(kTileThreads, kTileMinBlocks) gj_update_kernel(
    double* __restrict__ base, const long long* __restrict__ off, const int* __restrict__ ld,
    const int* __restrict__ n, int k, int symmetric, NextPivot nx, int pw, int compact) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  TileSmem& sm = *reinterpret_cast<TileSmem*>(smem_raw);
  const int b = blockIdx.y;
  const int nb = n[b];
  const int w = min(pw, nb - k);  // pivots of this step (panel width pw = 64 or 128)
  if (w <= 0) return;
  const int T = (nb + kTile - 1) / kTile;
  int tm, tn;
  if (compact) {
    // symmetric variant, compact grid: blockIdx.x enumerates only the lower-triangular
    // pairs (i >= j) of the tiles outside the pivot range (no CTAs that exit at once)
    const int x = blockIdx.x;
    int i = (int)((sqrtf(8.0f * (float)x + 1.0f) - 1.0f) * 0.5f);
    while ((i + 1) * (i + 2) / 2 <= x) ++i;
    while (i * (i + 1) / 2 > x) --i;
    const int j = x - i * (i + 1) / 2;
    const int ip = k / kTile, npv = pw / kTile;
    tm = i < ip ? i : i + npv;
    tn = j < ip ? j : j + npv;
  } else {
    tm = blockIdx.x / T;
    tn = blockIdx.x - tm * T;
  }
  if (tm >= T || tn >= T) return;
  const int r0 = tm * kTile, c0 = tn * kTile;
  if ((r0 >= k && r0 < k + pw) || (c0 >= k && c0 < k + pw)) return;
  if (symmetric && tn > tm) return;
  const int L = ld[b];
  double* M = base + off[b];
  double* Ct = (symmetric && tn < tm) ? M + (long long)c0 * L + r0 : nullptr;
  const double sgn = ((r0 < k) != (c0 < k)) ? -1.0 : 1.0;
  tile_mma(M + (long long)r0 * L + c0, L, min(kTile, nb - r0), min(kTile, nb - c0),
           M + (long long)r0 * L + k, L, M + (long long)k * L + c0, L, w, -1.0, 1.0, sm, Ct, L,
           sgn);
  if (nx.pinv != nullptr && r0 == k + kTile && c0 == k + kTile) {
    // lookahead: this CTA holds the next pivot block, final after this update
    __syncthreads();
    MmaGjSmem& gsm = *reinterpret_cast<MmaGjSmem*>(smem_raw);
    const bool bad = reg_gj64(M + (long long)r0 * L + r0, L, min(kTile, nb - r0),
                              nx.pinv + (long long)b * nx.stride, kTile, nx.require_positive,
                              nullptr, gsm);
    if (threadIdx.x == 0 && bad && nx.status)
      atomicCAS(nx.status + b, 0, nx.require_positive ? (int)kNotPositiveDefinite : (int)kSingularPivot);
  }
}

// M[r0 + r][k + c] = sgn * M[k + c][r0 + r] for r < h, c < w, transposed through
// shared memory (64 x 65 staging, 64 columns at a time) so that both the reads
// (rows of the row panel) and the writes (rows of the column panel) are coalesced
BDDC_DEV void gj_mirror_tile(double* M, long long L, int k, int w, int r0, int h, double sgn,
                             double* st) {
  for (int c0 = 0; c0 < w; c0 += kTile) {
    const int wc = min(kTile, w - c0);
    for (int idx = threadIdx.x; idx < h * wc; idx += blockDim.x) {
      const int c = idx / h, r = idx - c * h;
      st[c * 65 + r] = M[(long long)(k + c0 + c) * L + r0 + r];
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < h * wc; idx += blockDim.x) {
      const int r = idx / wc, c = idx - r * wc;
      M[(long long)(r0 + r) * L + k + c0 + c] = sgn * st[c * 65 + r];
    }
    __syncthreads();
  }
}

// ---- symmetric Gauss-Jordan in 128-wide panels (K = 128 trailing updates) ----
// pivot block of step k -> work (128 x 128, ld 128), identity beyond w
__global__ void gj128_extract_kernel(const double* __restrict__ base,
                                     const long long* __restrict__ off,
                                     const int* __restrict__ ld, const int* __restrict__ n, int k,
                                     double* __restrict__ work, int* __restrict__ work_n) {
  const int b = blockIdx.x;
  const int w = max(0, min(128, n[b] - k));
  // pivot blocks of at most 64 pivots are inverted by one register Gauss-Jordan
  // (pivot_inverse_kernel), whatever the rest of the batch needs: the work copy
  // is skipped (size 0), so every matrix takes the same route in any batch
  if (threadIdx.x == 0) work_n[b] = w > kTile ? 128 : 0;
  if (w <= kTile) return;
  const double* M = base + off[b] + (long long)k * ld[b] + k;
  double* W = work + (long long)b * 128 * 128;
  for (int idx = threadIdx.x; idx < 128 * 128; idx += blockDim.x) {
    const int r = idx >> 7, c = idx & 127;
    W[idx] = (r < w && c < w) ? M[(long long)r * ld[b] + c] : (r == c ? 1.0 : 0.0);
  }
}

// W = P A_(k, c0) in place (one 128 x 64 tile per CTA; BM = 128 so a single CTA
// owns every row it overwrites); the pivot column tiles receive sym(P)
__global__ void __launch_bounds__(512) gj128_row_kernel(double* __restrict__ base,
                                                        const long long* __restrict__ off,
                                                        const int* __restrict__ ld,
                                                        const int* __restrict__ n, int k,
                                                        const double* __restrict__ work) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  TileSmemT<128>& sm = *reinterpret_cast<TileSmemT<128>*>(smem_raw);
  const int b = blockIdx.y;
  const int nb = n[b];
  const int w = min(128, nb - k);
  if (w <= 0) return;
  const int c0 = blockIdx.x * kTile;
  if (c0 >= nb) return;
  const long long L = ld[b];
  double* M = base + off[b];
  const double* P = work + (long long)b * 128 * 128;
  if (c0 >= k && c0 < k + 128) {
    const int cc = c0 - k, wc = min(kTile, w - cc);
    for (int idx = threadIdx.x; idx < w * wc; idx += blockDim.x) {
      const int r = idx / wc, c = idx - r * wc;
      M[(long long)(k + r) * L + c0 + c] = 0.5 * (P[r * 128 + cc + c] + P[(cc + c) * 128 + r]);
    }
    return;
  }
  double* C = M + (long long)k * L + c0;
  tile_mma_t<128>(C, L, w, min(kTile, nb - c0), P, 128, C, L, w, 1.0, 0.0, sm);
}

// column panel of step k = +-(row panel)^T (symmetric variant)
__global__ void __launch_bounds__(kTileThreads, kTileMinBlocks) gj128_col_kernel(
    double* __restrict__ base, const long long* __restrict__ off, const int* __restrict__ ld,
    const int* __restrict__ n, int k) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int b = blockIdx.y;
  const int nb = n[b];
  const int w = min(128, nb - k);
  if (w <= 0) return;
  const int r0 = blockIdx.x * kTile;
  if (r0 >= nb || (r0 >= k && r0 < k + 128)) return;
  gj_mirror_tile(base + off[b], ld[b], k, w, r0, min(kTile, nb - r0), r0 < k ? 1.0 : -1.0,
                 reinterpret_cast<double*>(smem_raw));
}

__global__ void __launch_bounds__(kTileThreads, kTileMinBlocks) gj_col_kernel(
    double* __restrict__ base, const long long* __restrict__ off, const int* __restrict__ ld,
    const int* __restrict__ n, int k, const double* __restrict__ pinv, long long pinv_stride,
    int symmetric) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  TileSmem& sm = *reinterpret_cast<TileSmem*>(smem_raw);
  const int b = blockIdx.y;
  const int nb = n[b];
  const int w = min(kTile, nb - k);
  if (w <= 0) return;
  const int r0 = blockIdx.x * kTile;
  if (r0 >= nb) return;
  const int L = ld[b];
  double* M = base + off[b];
  const double* P = pinv + (long long)b * pinv_stride;
  if (r0 == k) {  // pivot block <- P (written by gj_row in the symmetric variant)
    if (symmetric) return;
    for (int idx = threadIdx.x; idx < w * w; idx += blockDim.x) {
      int r = idx / w, c = idx - r * w;
      M[(long long)(k + r) * L + k + c] =
          symmetric ? 0.5 * (P[r * kTile + c] + P[c * kTile + r]) : P[r * kTile + c];
    }
    return;
  }
  if (symmetric) {  // column panel = +-(row panel)^T: + for processed rows (G_KK), - for G_JK
    gj_mirror_tile(M, L, k, w, r0, min(kTile, nb - r0), r0 < k ? 1.0 : -1.0,
                   reinterpret_cast<double*>(smem_raw));
    return;
  }
  double* C = M + (long long)r0 * L + k;
  tile_mma(C, L, min(kTile, nb - r0), w, C, L, P, kTile, w, -1.0, 0.0, sm);
}

// ---------------------------------------------------------------------------
// extraction and small elementwise kernels
// ---------------------------------------------------------------------------
// S = M[nI:nL, nI:nL] -> S (ld nB), g = M[nI:nL, nL], Bsym = (S + S^T)/2.
// 32x32 tiles staged through shared memory so that both the tile and its
// transpose are read with coalesced rows (the transposed read of a naive
// element loop strides by ld).
__global__ void __launch_bounds__(256) extract_schur_kernel(
    const double* __restrict__ base, const long long* __restrict__ off,
    const int* __restrict__ ld, const int* __restrict__ nI, const int* __restrict__ nB,
    const long long* __restrict__ soff, const long long* __restrict__ voff,
    double* __restrict__ S, double* __restrict__ Bsym, double* __restrict__ g,
    double* __restrict__ s_norm2) {
  __shared__ double t0[32][33];
  __shared__ double t1[32][33];
  __shared__ double red[8];
  double sq = 0.0;
  const int b = blockIdx.y;
  const int n = nB[b], i0 = nI[b], L = ld[b];
  const double* M = base + off[b] + (long long)i0 * L + i0;
  double* Sb = S + soff[b];
  double* Bb = Bsym + soff[b];
  const int nt = (n + 31) / 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  for (int t = blockIdx.x; t < nt * nt; t += gridDim.x) {
    const int r0 = (t / nt) * 32, c0 = (t - (t / nt) * nt) * 32;
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 32; j += 8) {
      const int r = r0 + ty + j, c = c0 + tx;
      t0[ty + j][tx] = (r < n && c < n) ? M[(long long)r * L + c] : 0.0;
      const int rr = c0 + ty + j, cc = r0 + tx;  // transposed tile, read by rows
      t1[ty + j][tx] = (rr < n && cc < n) ? M[(long long)rr * L + cc] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 32; j += 8) {
      const int r = r0 + ty + j, c = c0 + tx;
      if (r < n && c < n) {
        const double v = t0[ty + j][tx];
        sq = fma(v, v, sq);
        Sb[(long long)r * n + c] = v;
        Bb[(long long)r * n + c] = 0.5 * (v + t1[tx][ty + j]);
      }
    }
  }
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x)
    g[voff[b] + r] = M[(long long)r * L + n];
  if (s_norm2 != nullptr) {  // this CTA's share of ||S_b||_F^2, fixed reduction tree
    for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
    __syncthreads();
    if (tx == 0) red[ty] = sq;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < 8; ++w) t += red[w];
      s_norm2[(long long)b * gridDim.x + blockIdx.x] = t;
    }
  }
}

// out[b] = sum of the kExtractParts partial sums of matrix b, in order
constexpr int kExtractParts = 48;
__global__ void sum_parts_kernel(const double* __restrict__ part, double* __restrict__ out,
                                 int nbatch) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nbatch) return;
  double t = 0.0;
  for (int x = 0; x < kExtractParts; ++x) t += part[(long long)b * kExtractParts + x];
  out[b] = t;
}

// out[b] = ||X_b||_F^2 for square batched matrices (ld = n); one CTA per
// matrix, fixed reduction tree (deterministic)
__global__ void __launch_bounds__(512) frob2_kernel(const double* __restrict__ X,
                                                    const long long* __restrict__ soff,
                                                    const int* __restrict__ nB,
                                                    double* __restrict__ out) {
  __shared__ double red[16];
  const int b = blockIdx.x;
  const long long nn = (long long)nB[b] * nB[b];
  const double* M = X + soff[b];
  double s = 0.0;
  for (long long idx = threadIdx.x; idx < nn; idx += blockDim.x) {
    const double v = M[idx];
    s = fma(v, v, s);
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    out[b] = t;
  }
}

// out[b] = trace(X_b)^2 (ld = n): for a symmetric positive definite X_b an upper
// bound of ||X_b||_F^2 (sum of squared eigenvalues <= squared sum) that reads
// only the diagonal; one warp per matrix, fixed reduction tree
__global__ void trace2_kernel(const double* __restrict__ X, const long long* __restrict__ soff,
                              const int* __restrict__ nB, double* __restrict__ out, int nbatch) {
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (b >= nbatch) return;
  const int n = nB[b], lane = threadIdx.x & 31;
  const double* M = X + soff[b];
  double s = 0.0;
  for (int i = lane; i < n; i += 32) s += M[(long long)i * (n + 1)];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[b] = s * s;
}

// X <- (X + X^T)/2 for square batched matrices (ld = n)
__global__ void symmetrize_kernel(double* __restrict__ X, const long long* __restrict__ soff,
                                  const int* __restrict__ nB) {
  const int b = blockIdx.y;
  const int n = nB[b];
  double* M = X + soff[b];
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < (long long)n * n;
       idx += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(idx / n), c = (int)(idx - (long long)r * n);
    if (c > r) {
      const double v = 0.5 * (M[(long long)r * n + c] + M[(long long)c * n + r]);
      M[(long long)r * n + c] = v;
      M[(long long)c * n + r] = v;
    }
  }
}

// ---------------------------------------------------------------------------
// interior recovery by block back-substitution over the stored W rows:
//   u_I[k:k+w] = Wf_k - W_k,(k+w:nL) u[k+w:nL]
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) recover_kernel(
    const double* __restrict__ base, const long long* __restrict__ off, const int* __restrict__ ld,
    const int* __restrict__ nI, const int* __restrict__ nB, const long long* __restrict__ voff,
    const int* __restrict__ iface_perm, const long long* __restrict__ ioff,
    const long long* __restrict__ interior_nodes, const double* __restrict__ u_hat,
    double* __restrict__ u, int panel, const int* __restrict__ ndeep) {
  extern __shared__ double us[];  // nI + nB
  const int b = blockIdx.x;
  const int ni = nI[b], nb = nB[b], L = ld[b], nl = ni + nb;
  const int nd = ndeep ? ndeep[b] : 0;
  const double* M = base + off[b];
  for (int j = threadIdx.x; j < nb; j += blockDim.x) us[ni + j] = u_hat[iface_perm[voff[b] + j]];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  // panels of the elimination (W = A11^-1 A12 per panel, identity diagonal):
  // second phase (pivots [nd, ni), panels from nd) first, then the deep pivots
  // [0, nd), whose rows have no entries in the interface columns
  for (int phase = 1; phase >= 0; --phase) {
    const int p0 = phase ? nd : 0, p1 = phase ? ni : nd;
    if (p1 <= p0) continue;
    const int cend = phase ? nl : ni;
    const int last = p0 + ((p1 - p0 - 1) / panel) * panel;
    for (int k = last; k >= p0; k -= panel) {
      const int w = min(panel, p1 - k);
      for (int r = k + warp; r < k + w; r += nw) {
        const double* row = M + (long long)r * L;
        double s = 0.0;
        for (int c = k + w + lane; c < cend; c += 32) s += row[c] * us[c];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) us[r] = row[nl] - s;
      }
      __syncthreads();
    }
  }
  for (int j = threadIdx.x; j < ni; j += blockDim.x) u[interior_nodes[ioff[b] + j]] = us[j];
}

}  // namespace bddc

// ===========================================================================
// C-ABI
// ===========================================================================
using namespace bddc;

static int smem_tile_setup() {
  static PerDeviceOnce once;
  once([&] {
    int bytes = (int)sizeof(TileSmem);
    cudaFuncSetAttribute(schur_row_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    cudaFuncSetAttribute(schur_trailing_kernel<kTrailBM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(TileSmemT<kTrailBM>));
    cudaFuncSetAttribute(schur_trailing_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(TileSmemT<64>));
    cudaFuncSetAttribute(gj_row_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    cudaFuncSetAttribute(gj_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    cudaFuncSetAttribute(gj_col_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    cudaFuncSetAttribute(panel_scale_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  });
  return (int)sizeof(TileSmem);
}

static int launch_status() {
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : -(int)e;
}

extern "C" {

int bddc_plan_loc4(const long long* conn, const long long* sub_of, long long n_elements, int s0,
                   const int* iloc_of_node, const int* glob_of_node, const int* pos_in_glob,
                   const int* sh_start, const int* sh_sub, const int* sh_boff,
                   const long long* nI, int* loc4, cudaStream_t stream) {
  if (n_elements <= 0) return 0;
  const long long nc = 4 * n_elements;
  const int grid = (int)((nc + 255) / 256 < 148 * 16 ? (nc + 255) / 256 : 148 * 16);
  plan_loc4_kernel<<<grid, 256, 0, stream>>>(conn, sub_of, nc, s0, iloc_of_node, glob_of_node,
                                             pos_in_glob, sh_start, sh_sub, sh_boff, nI, loc4);
  bddc_note_launches(1);
  return launch_status();
}

int bddc_local_assemble(double* K, const long long* off, const int* ld, const int* nloc,
                        const long long* elem_start, const long long* elem_ids, const int* loc4,
                        const long long* conn, const double* Ke, const double* Fe,
                        const double* gdir, int nbatch, int max_nl, int* lists, long long* keys,
                        int* overflow, int general, const int* nint, const int* ndeep,
                        cudaStream_t stream) {
  if (nbatch <= 0) return 0;
  int nrowbuf = 0;  // compact row phase (row lists + one row buffer per warp)
  if (general) {
    nrowbuf = kAsmWarps;
    while (nrowbuf > 1 && assemble_smem_bytes(max_nl, nrowbuf) > 200 * 1024) --nrowbuf;
  }
  const size_t smem = assemble_smem_bytes(max_nl, nrowbuf);
  if (smem > 227 * 1024) return -(int)cudaErrorInvalidValue;
  cudaFuncSetAttribute(assemble_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  assemble_rows_kernel<<<nbatch, kAsmWarps * 32, smem, stream>>>(
      K, off, ld, nloc, elem_start, elem_ids, loc4, conn, Ke, Fe, gdir, lists, keys, nrowbuf,
      overflow, (int)assemble_region0(max_nl, nrowbuf), nint, ndeep);
  bddc_note_launches(1);
  return launch_status();
}

// Optional event log of the trailing-update launches (bench roofline over the
// timed region without a mid-step synchronisation): bddc_trailing_log(1)
// starts it, bddc_trailing_collect() sums the logged durations and clears it.
// per host thread (the C-ABI keeps no process-wide mutable state besides the
// launch counter): each thread driving a device has its own log
static thread_local std::vector<cudaEvent_t> g_trail_pool;  // created once, reused
static thread_local size_t g_trail_used = 0;
static thread_local bool g_trail_on = false;

static int schur_eliminate_impl(double* M, const long long* off, const int* ld, const int* npiv,
                                const int* nrows, const int* ncols, int nbatch, int max_npiv,
                                int max_rows, int max_cols, int panel, double* pinv_ws,
                                long long pinv_stride, long long pinv_step_stride, int* status,
                                int require_positive, double* piv_out, long long piv_stride,
                                const int* hole0, const int* hole1, cudaStream_t stream,
                                double* host_trailing_ms) {
  if (nbatch <= 0) return 0;
  if (panel != 2 * kTile) panel = kTile;
  const ColHole hole{hole0, hole0 ? hole1 : nullptr};
  const int smem = smem_tile_setup();
  const int nsteps = (max_npiv + panel - 1) / panel;
  cudaEvent_t* ev = nullptr;
  if (host_trailing_ms) {
    ev = new cudaEvent_t[2 * nsteps];
    for (int i = 0; i < 2 * nsteps; ++i) cudaEventCreate(&ev[i]);
    *host_trailing_ms = 0.0;
  }
  int launches = 0, timed = 0;
  const size_t tsm = sizeof(TileSmemT<kTrailBM>);
  const NextPivot none{nullptr, 0, nullptr, 0, nullptr, 0};
  // pivot blocks after the first are inverted inside the launch that last
  // updates them (lookahead); pivoted[k / 64] tracks which were
  pivot_inverse_kernel<<<nbatch, 256, 0, stream>>>(M, off, ld, npiv, 0, pinv_ws, pinv_stride,
                                                   status, require_positive, piv_out, piv_stride);
  ++launches;
  for (int k = 0; k < max_npiv; k += panel) {
    // pivot inverses are kept per 64-wide sub-panel (step stride per 64 pivots)
    double* P = pinv_ws + (long long)(k / kTile) * pinv_step_stride;
    double* P2 = pinv_ws + (long long)(k / kTile + 1) * pinv_step_stride;
    double* Pn = pinv_ws + (long long)((k + panel) / kTile) * pinv_step_stride;
    const NextPivot nx_sub{P2, pinv_stride, status, require_positive, piv_out, piv_stride};
    const NextPivot nx_next{Pn, pinv_stride, status, require_positive, piv_out, piv_stride};
    bool next_done = false;
    // first (or only) 64-wide sub-panel: W1 = P1 A12 (P1 from the previous launch)
    const int ct1 = ceil_div(max_cols - k, kTile);
    if (ct1 > 0) {
      schur_row_kernel<<<dim3(ct1, nbatch), kTileThreads, smem, stream>>>(
          M, off, ld, npiv, ncols, k, P, pinv_stride, 0x7fffffff, hole);
      ++launches;
    }
    if (panel == 2 * kTile && k + kTile < max_npiv) {
      // second sub-panel: the K = 64 update by the first one on its 64 rows (+ its
      // pivot inverse) and on its column panel below the 128-wide panel, then W2
      const int cts = ceil_div(max_cols - k - kTile, kTile);
      // (column-panel tiles start at row k + w_b >= k + 65 of each matrix: bound for all)
      const int rts = max(0, ceil_div(max_rows - k - kTile, kTile));
      schur_trailing_kernel<64><<<dim3(cts + rts, nbatch), kTileThreads, sizeof(TileSmemT<64>),
                                  stream>>>(M, off, ld, npiv, nrows, ncols, k, 0x7fffffff, kTile, 1,
                                            nx_sub, hole);
      schur_row_kernel<<<dim3(cts, nbatch), kTileThreads, smem, stream>>>(
          M, off, ld, npiv, ncols, k + kTile, P2, pinv_stride, 0x7fffffff, hole);
      launches += 2;
    }
    const int ct = ceil_div(max_cols - k, kTile);
    const int rt = ceil_div(max_rows - k, kTrailBM);
    const bool more = k + panel < max_npiv;
    if (ct > 0 && rt > 0) {
      const bool lg = g_trail_on && !ev && g_trail_used + 2 <= g_trail_pool.size();
      if (lg) cudaEventRecord(g_trail_pool[g_trail_used], stream);
      if (ev) cudaEventRecord(ev[2 * timed], stream);
      schur_trailing_kernel<kTrailBM><<<dim3(ct * rt, nbatch), kTrailBM * 4, tsm, stream>>>(
          M, off, ld, npiv, nrows, ncols, k, 0x7fffffff, panel, 0, more ? nx_next : none, hole);
      ++launches;
      next_done = true;
      if (ev) cudaEventRecord(ev[2 * timed + 1], stream);
      if (lg) {
        cudaEventRecord(g_trail_pool[g_trail_used + 1], stream);
        g_trail_used += 2;
      }
      timed += (ev != nullptr);
    }
    if (more && !next_done) {
      pivot_inverse_kernel<<<nbatch, 256, 0, stream>>>(M, off, ld, npiv, k + panel, Pn, pinv_stride,
                                                       status, require_positive, piv_out,
                                                       piv_stride);
      ++launches;
    }
  }
  if (ev) {
    if (timed) cudaEventSynchronize(ev[2 * timed - 1]);
    for (int i = 0; i < timed; ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[2 * i], ev[2 * i + 1]);
      *host_trailing_ms += ms;
    }
    for (int i = 0; i < 2 * nsteps; ++i) cudaEventDestroy(ev[i]);
    delete[] ev;
  }
  bddc_note_launches(launches);
  return launch_status();
}

int bddc_schur_eliminate(double* M, const long long* off, const int* ld, const int* npiv,
                         const int* nrows, const int* ncols, int nbatch, int max_npiv,
                         int max_rows, int max_cols, int panel, double* pinv_ws,
                         long long pinv_stride, long long pinv_step_stride, int* status,
                         int require_positive, double* piv_out, long long piv_stride,
                         const int* col_hole0, const int* col_hole1, cudaStream_t stream) {
  return schur_eliminate_impl(M, off, ld, npiv, nrows, ncols, nbatch, max_npiv, max_rows,
                              max_cols, panel, pinv_ws, pinv_stride, pinv_step_stride, status,
                              require_positive, piv_out, piv_stride, col_hole0, col_hole1, stream,
                              nullptr);
}

int bddc_trailing_log(int enable) {
  if (enable && g_trail_pool.empty()) {
    g_trail_pool.resize(4096);
    for (cudaEvent_t& e : g_trail_pool) cudaEventCreate(&e);
  }
  g_trail_on = enable != 0;
  return 0;
}

int bddc_trailing_collect(double* total_ms, long long* launches) {
  double t = 0.0;
  for (size_t i = 0; i + 1 < g_trail_used; i += 2) {
    float ms = 0.f;
    cudaEventSynchronize(g_trail_pool[i + 1]);
    cudaEventElapsedTime(&ms, g_trail_pool[i], g_trail_pool[i + 1]);
    t += ms;
  }
  *total_ms = t;
  *launches = (long long)(g_trail_used / 2);
  g_trail_used = 0;
  return 0;
}

int bddc_schur_eliminate_timed(double* M, const long long* off, const int* ld, const int* npiv,
                               const int* nrows, const int* ncols, int nbatch, int max_npiv,
                               int max_rows, int max_cols, int panel, double* pinv_ws,
                               long long pinv_stride, long long pinv_step_stride, int* status,
                               int require_positive, double* piv_out, long long piv_stride,
                               const int* col_hole0, const int* col_hole1, cudaStream_t stream,
                               double* host_trailing_ms) {
  return schur_eliminate_impl(M, off, ld, npiv, nrows, ncols, nbatch, max_npiv, max_rows,
                              max_cols, panel, pinv_ws, pinv_stride, pinv_step_stride, status,
                              require_positive, piv_out, piv_stride, col_hole0, col_hole1, stream,
                              host_trailing_ms);
}

int bddc_gj_inverse(double* M, const long long* off, const int* ld, const int* n, int nbatch,
                    int max_n, double* pinv_ws, long long pinv_stride, int* status,
                    int require_positive, int symmetric, cudaStream_t stream) {
  if (nbatch <= 0) return 0;
  const int smem = smem_tile_setup();
  const int T = ceil_div(max_n, kTile);
  const NextPivot none{nullptr, 0, nullptr, 0, nullptr, 0};
  const bool look = symmetric != 0;
  const NextPivot nx{pinv_ws, pinv_stride, status, require_positive, nullptr, 0};
  for (int k = 0; k < max_n; k += kTile) {
    // symmetric: pivots after the first are inverted by the update launch (lookahead)
    if (!look || k == 0) {
      pivot_inverse_kernel<<<nbatch, 256, 0, stream>>>(M, off, ld, n, k, pinv_ws, pinv_stride,
                                                       status, require_positive, nullptr, 0);
      bddc_note_launches(1);
    }
    gj_row_kernel<<<dim3(T, nbatch), kTileThreads, smem, stream>>>(M, off, ld, n, k, pinv_ws,
                                                                  pinv_stride, symmetric);
    if (symmetric) {  // lower-triangular pairs of the T - 1 tiles outside the pivot tile
      const int na = T - 1;
      if (na > 0)
        gj_update_kernel<<<dim3(na * (na + 1) / 2, nbatch), kTileThreads, smem, stream>>>(
            M, off, ld, n, k, 1, look && k + kTile < max_n ? nx : none, kTile, 1);
    } else {
      gj_update_kernel<<<dim3(T * T, nbatch), kTileThreads, smem, stream>>>(M, off, ld, n, k, 0, none,
                                                                           kTile, 0);
    }
    gj_col_kernel<<<dim3(T, nbatch), kTileThreads, smem, stream>>>(M, off, ld, n, k, pinv_ws,
                                                                  pinv_stride, symmetric);
    bddc_note_launches(3);
  }
  return launch_status();
}

int bddc_gj_inverse128(double* M, const long long* off, const int* ld, const int* n, int nbatch,
                       int max_n, double* work, const long long* work_off, const int* work_ld,
                       int* work_n, double* pinv_ws, int* status, int require_positive,
                       cudaStream_t stream) {
  if (nbatch <= 0) return 0;
  const int smem = smem_tile_setup();
  static PerDeviceOnce once;
  once([&] {
    cudaFuncSetAttribute(gj128_row_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(TileSmemT<128>));
    cudaFuncSetAttribute(gj128_col_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  });
  const int T = ceil_div(max_n, kTile);
  const NextPivot none{nullptr, 0, nullptr, 0, nullptr, 0};
  for (int k = 0; k < max_n; k += 128) {
    // panels of at most 64 pivots (the last one of a matrix): the inverse straight
    // into the work block (leading dimension 128) by one register Gauss-Jordan
    pivot_inverse_kernel<<<nbatch, 256, 0, stream>>>(M, off, ld, n, k, work, 128 * 128, status,
                                                     require_positive, nullptr, 0, 128, 1);
    bddc_note_launches(1);
    if (max_n - k > kTile) {
      gj128_extract_kernel<<<nbatch, 256, 0, stream>>>(M, off, ld, n, k, work, work_n);
      bddc_note_launches(1);
      // P = (pivot block)^-1: symmetric 64-panel Gauss-Jordan on the 128 x 128 copies
      // (positive LDL^T pivots <=> positive definite: the cho_factor criterion)
      int rc = bddc_gj_inverse(work, work_off, work_ld, work_n, nbatch, 128, pinv_ws, 4096, status,
                               require_positive, 1, stream);
      if (rc) return rc;
    }
    gj128_row_kernel<<<dim3(T, nbatch), 512, sizeof(TileSmemT<128>), stream>>>(M, off, ld, n, k,
                                                                               work);
    {  // lower-triangular pairs of the tiles outside the (up to two) pivot tiles
      const int na = T - min(2, T - k / kTile);
      if (na > 0)
        gj_update_kernel<<<dim3(na * (na + 1) / 2, nbatch), kTileThreads, smem, stream>>>(
            M, off, ld, n, k, 1, none, 128, 1);
    }
    gj128_col_kernel<<<dim3(T, nbatch), kTileThreads, smem, stream>>>(M, off, ld, n, k);
    bddc_note_launches(3);
  }
  return launch_status();
}

int bddc_extract_schur(const double* M, const long long* off, const int* ld, const int* nI,
                       const int* nB, const long long* soff, const long long* voff, double* S,
                       double* Bsym, double* g, int nbatch, double* s_norm2, double* norm_ws,
                       cudaStream_t stream) {
  if (nbatch <= 0) return 0;
  const bool norms = s_norm2 != nullptr && norm_ws != nullptr;
  extract_schur_kernel<<<dim3(kExtractParts, nbatch), 256, 0, stream>>>(
      M, off, ld, nI, nB, soff, voff, S, Bsym, g, norms ? norm_ws : nullptr);
  bddc_note_launches(1);
  if (norms) {
    sum_parts_kernel<<<ceil_div(nbatch, 256), 256, 0, stream>>>(norm_ws, s_norm2, nbatch);
    bddc_note_launches(1);
  }
  return launch_status();
}

int bddc_frob2(const double* X, const long long* soff, const int* n, int nbatch, double* out,
               cudaStream_t stream) {
  if (nbatch <= 0) return 0;
  frob2_kernel<<<nbatch, 512, 0, stream>>>(X, soff, n, out);
  bddc_note_launches(1);
  return launch_status();
}

int bddc_trace2(const double* X, const long long* soff, const int* n, int nbatch, double* out,
                cudaStream_t stream) {
  if (nbatch <= 0) return 0;
  trace2_kernel<<<ceil_div(nbatch, 8), 256, 0, stream>>>(X, soff, n, out, nbatch);
  bddc_note_launches(1);
  return launch_status();
}

int bddc_symmetrize(double* X, const long long* soff, const int* n, int nbatch,
                    cudaStream_t stream) {
  if (nbatch <= 0) return 0;
  symmetrize_kernel<<<dim3(64, nbatch), 256, 0, stream>>>(X, soff, n);
  bddc_note_launches(1);
  return launch_status();
}

int bddc_recover_interior(const double* M, const long long* off, const int* ld, const int* nI,
                          const int* nB, const long long* voff, const int* iface_perm,
                          const long long* ioff, const long long* interior_nodes,
                          const double* u_hat, double* u, int nbatch, int max_nloc, int panel,
                          const int* ndeep, cudaStream_t stream) {
  if (nbatch <= 0) return 0;
  const int smem = max_nloc * (int)sizeof(double);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(recover_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  recover_kernel<<<nbatch, 256, smem, stream>>>(M, off, ld, nI, nB, voff, iface_perm, ioff,
                                                interior_nodes, u_hat, u, panel, ndeep);
  bddc_note_launches(1);
  return launch_status();
}

}  // extern "C"
