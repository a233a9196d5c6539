// Low-rank SI-DSA on the GPU: LowRankBasis (CGS with conditional second
// pass and overlap-triggered Householder rebuild, border-extended
// projections), greedy residual subsampling, the inner loop and the outer
// driver (proj/src/low_rank.cpp:39-492).
//
// The control flow, the RNG (mt19937_64 + masked rejection) and every gate
// stay on the host exactly as in the reference; every O(N_x) or O(r^3)
// operation runs on the device: sweeps (K1), CGS GEMVs (K4), the streaming
// stencils of the border extension (K5), the X^T [W | rhs] GEMM (K6), the
// batched Galerkin LU solves (K7), X C expansion + fused residual norms
// (K8/K3), phi = X (C w) (K10), QR / Jacobi SVD (K11) and the DSA (K12).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <numeric>
#include <cstdlib>
#include <cstdio>
#include <string>

#include <cooperative_groups.h>

#include "dense.cuh"
#include "lowrank.hpp"
#include "problem.hpp"

namespace rtlr {
namespace cuda {

namespace {

__global__ void proj_border_kernel(int r0, int pn, int pchunk_off, int pc, const double* __restrict__ G, long long ldg,
                                   double* __restrict__ proj, long long ldp, long long pstride, int rtot) {
  // G = X[:, 0:rtot]^T [Dx-P, Dx-^T P, Dy-P, Dy-^T P, St P] for the pc new
  // columns r0+pchunk_off .. r0+pchunk_off+pc-1 (column j of block k at k*pc+j).
  const long long total = static_cast<long long>(rtot) * pc;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(e % rtot), j = static_cast<int>(e / rtot);
    const int col = r0 + pchunk_off + j;
    const double g0 = G[i + (0 * pc + j) * ldg], g1 = G[i + (1 * pc + j) * ldg];
    const double g2 = G[i + (2 * pc + j) * ldg], g3 = G[i + (3 * pc + j) * ldg];
    const double g4 = G[i + (4 * pc + j) * ldg];
    // column `col` of every projection: X^T A x_col
    proj[i + col * ldp + 0 * pstride] = g0;   // Dx^-
    proj[i + col * ldp + 1 * pstride] = -g1;  // Dx^+ = -(Dx^-)^T
    proj[i + col * ldp + 2 * pstride] = g2;
    proj[i + col * ldp + 3 * pstride] = -g3;
    proj[i + col * ldp + 4 * pstride] = g4;
    // row `col` restricted to the old columns i < r0: x_col^T A x_i =
    // (A^T x_col)^T x_i
    if (i < r0) {
      proj[col + i * ldp + 0 * pstride] = g1;
      proj[col + i * ldp + 1 * pstride] = -g0;
      proj[col + i * ldp + 2 * pstride] = g3;
      proj[col + i * ldp + 3 * pstride] = -g2;
      proj[col + i * ldp + 4 * pstride] = g4;
    }
  }
}

__global__ void scatter_cols(int r, int m, const int* __restrict__ idx, const double* __restrict__ src, long long lds,
                             double* __restrict__ dst, long long ldd) {
  const long long total = static_cast<long long>(r) * m;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(e % r), j = static_cast<int>(e / r);
    dst[i + idx[j] * ldd] = src[i + j * lds];
  }
}

__global__ void gather_cols(int r, int m, const int* __restrict__ idx, const double* __restrict__ src, long long lds,
                            double* __restrict__ dst, long long ldd) {
  const long long total = static_cast<long long>(r) * m;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(e % r), j = static_cast<int>(e / r);
    dst[i + j * ldd] = src[i + idx[j] * lds];
  }
}

__global__ void transpose_kernel(int rows, int cols, const double* __restrict__ a, long long lda,
                                 double* __restrict__ b, long long ldb) {
  const long long total = static_cast<long long>(rows) * cols;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(e % rows), j = static_cast<int>(e / rows);
    b[j + i * ldb] = a[i + j * lda];
  }
}

__global__ void col_norms_kernel(long long m, int n, const double* __restrict__ w, long long ldw, double* out) {
  __shared__ double sh[32];
  const int j = blockIdx.x;
  double s = 0.0;
  for (long long i = threadIdx.x; i < m; i += blockDim.x) s += w[i + j * ldw] * w[i + j * ldw];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < (blockDim.x >> 5); ++k) t += sh[k];
    out[j] = sqrt(t);
  }
}

// The CGS batch's remainder copy Rm = S and the snapshots' norms in one
// pass over S: grid (kSnapParts, columns), each CTA a contiguous row chunk
// (fixed-order partials, 16-byte loads), then one warp per column sums the
// partials in a fixed order.  (The column-per-CTA kernel above used only p
// CTAs: 600 us per C4 batch for 64 MB.)
constexpr int kSnapParts = 128;
__global__ void __launch_bounds__(256) copy_norm_parts(long long m, const double* __restrict__ w, long long ldw,
                                                       double* __restrict__ dst, long long ldd,
                                                       double* __restrict__ part) {
  __shared__ double sh[8];
  const int j = blockIdx.y;
  const long long pairs = m >> 1;
  const long long per = (pairs + kSnapParts - 1) / kSnapParts;
  const long long q0 = blockIdx.x * per, q1 = min(pairs, q0 + per);
  const double* c = w + j * ldw;
  double* d = dst ? dst + j * ldd : nullptr;
  const bool vec = ((ldw | ldd) & 1) == 0 && (reinterpret_cast<uintptr_t>(w) & 15) == 0 &&
                   (!dst || (reinterpret_cast<uintptr_t>(dst) & 15) == 0);
  double s = 0.0;
  for (long long q = q0 + threadIdx.x; q < q1; q += blockDim.x) {
    double2 v;
    if (vec) {
      v = reinterpret_cast<const double2*>(c)[q];
      if (d) reinterpret_cast<double2*>(d)[q] = v;
    } else {
      v.x = c[2 * q];
      v.y = c[2 * q + 1];
      if (d) {
        d[2 * q] = v.x;
        d[2 * q + 1] = v.y;
      }
    }
    s += v.x * v.x;
    s += v.y * v.y;
  }
  if (blockIdx.x == kSnapParts - 1 && (m & 1) && threadIdx.x == 0) {
    const double v = c[m - 1];
    if (d) d[m - 1] = v;
    s += v * v;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < 8; ++k) t += sh[k];
    part[static_cast<size_t>(j) * kSnapParts + blockIdx.x] = t;
  }
}

__global__ void norm_parts_finish(int n, const double* __restrict__ part, double* __restrict__ out) {
  const int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (j >= n) return;
  double s = 0.0;
  for (int k = lane; k < kSnapParts; k += 32) s += part[static_cast<size_t>(j) * kSnapParts + k];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[j] = sqrt(s);
}

__global__ void scale_val_kernel(long long n, const double* __restrict__ x, double h, double* __restrict__ y) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    y[i] = x[i] / h;
}

__global__ void add_vec(int n, double* __restrict__ a, const double* __restrict__ b) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a[i] += b[i];
}

__global__ void sqdiff_partials(long long rows, int cols, const double* __restrict__ a, long long lda,
                                const double* __restrict__ b, long long ldb, double* __restrict__ part) {
  // part[blockIdx.x] = sum over this block's fixed share of (a - b)^2
  __shared__ double sh[32];
  const long long total = rows * cols;
  double s = 0.0;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long i = e % rows, j = e / rows;
    const double d = a[i + j * lda] - b[i + j * ldb];
    s += d * d;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < (blockDim.x >> 5); ++k) t += sh[k];
    part[blockIdx.x] = t;
  }
}

// ---- the within-batch CGS of mgs_ro_update on the device, no host syncs:
// the accepted count k, the second-pass flag, h and the accept/position
// flags live in device memory and gate the kernels; the host reads the
// batch's outcome once (low_rank.cpp:74-105).
constexpr int kCgsMax = 16;     // snapshots per batch handled on the device
constexpr int kCgsParts = 296;  // fixed row partition of the dot products

struct CgsState {
  int k;                  // vectors accepted so far in this batch
  int do2;                // second pass for the current snapshot
  int acc[kCgsMax], pos[kCgsMax];
  double rn2, h2;         // |rem|^2 after pass 1 / after all passes
  double h[kCgsMax];
  double coef[kCgsMax][kCgsMax];  // coef[i][j] = x_{r_old+j}^T rem_i (both passes)
  double c[kCgsMax];      // the current pass's coefficients
  int ocol;               // last accepted column when the overlap test applies, else -1
  double overlap;         // x_0^T x_ocol (low_rank.cpp:107-111)
};

// partial dots of X[:, j] (j < min(m, st.k)) with v; part[j * gridDim.x + block]
__global__ void __launch_bounds__(256) cgs_dots(long long n, int m, const double* __restrict__ X, long long ldx,
                                                const double* __restrict__ v, const CgsState* st, bool second,
                                                double* __restrict__ part) {
  __shared__ double sh[8][kCgsMax];
  if (second && !st->do2) return;
  const int k = min(m, st->k);
  if (k == 0) return;
  double acc[kCgsMax];
#pragma unroll
  for (int j = 0; j < kCgsMax; ++j) acc[j] = 0.0;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const double vi = v[i];
#pragma unroll
    for (int j = 0; j < kCgsMax; ++j)
      if (j < k) acc[j] += X[i + j * ldx] * vi;
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < kCgsMax; ++j) {
    double t = acc[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) sh[w][j] = t;
  }
  __syncthreads();
  if (threadIdx.x < k) {
    double t = 0.0;
    for (int ww = 0; ww < (blockDim.x >> 5); ++ww) t += sh[ww][threadIdx.x];
    part[threadIdx.x * gridDim.x + blockIdx.x] = t;
  }
}

// c[j] = sum of the partials in block order; coef[i][j] += c[j]; one warp per j
__global__ void cgs_finish(int m, int parts, const double* __restrict__ part, CgsState* st, int i, bool second) {
  if (second && !st->do2) return;
  const int k = min(m, st->k);
  const int j = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (j >= k) return;
  double t = 0.0;
  for (int z = lane; z < parts; z += 32) t += part[j * parts + z];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if (lane == 0) {
    st->c[j] = t;
    st->coef[i][j] += t;
  }
}

// v -= X[:, 0:k] c
__global__ void cgs_axpy(long long n, int m, const double* __restrict__ X, long long ldx, const CgsState* st,
                         bool second, double* __restrict__ v) {
  if (second && !st->do2) return;
  const int k = min(m, st->k);
  if (k == 0) return;
  double c[kCgsMax];
#pragma unroll
  for (int j = 0; j < kCgsMax; ++j) c[j] = j < k ? st->c[j] : 0.0;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < kCgsMax; ++j)
      if (j < k) s += X[i + j * ldx] * c[j];
    v[i] -= s;
  }
}

// the reference's conditional second pass: |rem| < 0.5 |snapshot| after pass 1
__global__ void cgs_gate(CgsState* st, const double* norm0p) {
  const double norm0 = *norm0p;
  st->do2 = st->k > 0 && sqrt(st->rn2) < 0.5 * norm0;
}

// drop test h > 1e-12 |snapshot| (low_rank.hpp:61-62): accepted vectors take
// the next column
__global__ void cgs_accept(CgsState* st, int i, const double* norm0p, double drop_tol) {
  const double norm0 = *norm0p;
  const double h = sqrt(st->h2);
  st->h[i] = h;
  const int acc = norm0 > 0.0 && h > drop_tol * norm0;
  st->acc[i] = acc;
  st->pos[i] = st->k;
  if (acc) ++st->k;
}

__global__ void cgs_store(long long n, const double* __restrict__ v, const CgsState* st, int i,
                          double* __restrict__ X0, long long ldx) {
  if (!st->acc[i]) return;
  double* col = X0 + static_cast<long long>(st->pos[i]) * ldx;
  const double h = st->h[i];
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<long long>(gridDim.x) * blockDim.x)
    col[e] = v[e] / h;
}

// The batch's record columns (low_rank.cpp:96-104) straight into the device
// record: old-basis coefficients (both block passes, summed as the host did),
// this batch's within-batch coefficients, h when accepted.  Column i of the
// batch at rec + i*ldr; rows beyond a column's length stay zero.
__global__ void rec_batch_kernel(int r_old, int p_in, const double* __restrict__ C1, const double* __restrict__ C2,
                                 const CgsState* __restrict__ st, double* __restrict__ rec, long long ldr) {
  const int i = blockIdx.x;
  if (i >= p_in) return;
  double* col = rec + static_cast<long long>(i) * ldr;
  const int kb = st->pos[i];
  for (int k = threadIdx.x; k < r_old; k += blockDim.x)
    col[k] = C1[k + static_cast<long long>(i) * r_old] + C2[k + static_cast<long long>(i) * r_old];
  for (int j = threadIdx.x; j < kb; j += blockDim.x) col[r_old + j] = st->coef[i][j];
  if (threadIdx.x == 0 && st->acc[i]) col[r_old + kb] = st->h[i];
}

// The overlap test's column (low_rank.cpp:107-111): only when this batch
// added a column and the rank is >= 2.
__global__ void overlap_col_kernel(CgsState* st, int r_old) {
  const int r = r_old + st->k;
  st->ocol = (st->k > 0 && r >= 2) ? r - 1 : -1;
  st->overlap = 0.0;
}

// The whole within-batch CGS of one batch in one cooperative launch
// (kCgsParts CTAs x 256 threads, grid-wide barriers between dependent
// steps) instead of ~13 launches per snapshot.  Every CTA reduces the
// partials itself, in the order cgs_finish / dot_finish use, and the
// per-thread index sets are those of cgs_dots / dot_partials, so the
// results (and the CgsState the host reads) are bitwise those of the
// launch-per-step sequence above.
__device__ __forceinline__ double cgs_warp_sum(double t) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  return t;
}

__global__ void __launch_bounds__(256, 2) cgs_batch_kernel(long long n, int p_in, const double* __restrict__ norm0,
                                                           double drop_tol,
                                                           double* __restrict__ R,
                                                           double* __restrict__ X, long long ldx, CgsState* st,
                                                           double* __restrict__ part, double* __restrict__ part2) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ double sh[8][kCgsMax];
  __shared__ double csh[kCgsMax];
  __shared__ double red[8];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  const long long i0 = blockIdx.x * static_cast<long long>(blockDim.x) + tid;
  const bool lead = blockIdx.x == 0;
  // sum over the kCgsParts partials part2[] as dot_finish does (one block of 256)
  auto finish_dot = [&]() -> double {
    double v = 0.0;
    for (int z = tid; z < static_cast<int>(gridDim.x); z += blockDim.x) v += part2[z];
    v = cgs_warp_sum(v);
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    double t = 0.0;
    for (int ww = 0; ww < 8; ++ww) t += red[ww];
    __syncthreads();
    return t;
  };
  // this CTA's partial of sum v^2 (block_sum_all order) into part2[block]
  auto store_norm_partial = [&](double sv) {
    sv = cgs_warp_sum(sv);
    __syncthreads();
    if (lane == 0) red[w] = sv;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int ww = 0; ww < 8; ++ww) t += red[ww];
      part2[blockIdx.x] = t;
    }
    __syncthreads();
  };
  // one projection pass of v against X[:, 0:k]: dots, reduction, v -= X c
  // fused with the partial of |v|^2; coef[i][:] += c
  auto pass = [&](double* v, int k, int i) {
    double acc[kCgsMax];
#pragma unroll
    for (int j = 0; j < kCgsMax; ++j) acc[j] = 0.0;
    for (long long e = i0; e < n; e += stride) {
      const double vi = v[e];
#pragma unroll
      for (int j = 0; j < kCgsMax; ++j)
        if (j < k) acc[j] += X[e + j * ldx] * vi;
    }
#pragma unroll
    for (int j = 0; j < kCgsMax; ++j) {
      const double t = cgs_warp_sum(acc[j]);
      if (lane == 0) sh[w][j] = t;
    }
    __syncthreads();
    if (tid < k) {
      double t = 0.0;
      for (int ww = 0; ww < 8; ++ww) t += sh[ww][tid];
      part[tid * gridDim.x + blockIdx.x] = t;
    }
    grid.sync();
    for (int j = w; j < k; j += 8) {  // cgs_finish's order: lanes stride the partials, xor tree
      double t = 0.0;
      for (int z = lane; z < static_cast<int>(gridDim.x); z += 32) t += part[j * gridDim.x + z];
      t = cgs_warp_sum(t);
      if (lane == 0) csh[j] = t;
    }
    __syncthreads();
    if (lead && tid < k) {
      st->c[tid] = csh[tid];
      st->coef[i][tid] += csh[tid];
    }
    double c[kCgsMax];
#pragma unroll
    for (int j = 0; j < kCgsMax; ++j) c[j] = j < k ? csh[j] : 0.0;
    double sv = 0.0;
    for (long long e = i0; e < n; e += stride) {
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < kCgsMax; ++j)
        if (j < k) s += X[e + j * ldx] * c[j];
      const double nv = v[e] - s;
      v[e] = nv;
      sv += nv * nv;
    }
    store_norm_partial(sv);
    grid.sync();
  };
  auto norm_only = [&](const double* v) {
    double sv = 0.0;
    for (long long e = i0; e < n; e += stride) sv += v[e] * v[e];
    store_norm_partial(sv);
    grid.sync();
  };
  int k = 0;
  for (int i = 0; i < p_in; ++i) {
    double* rem = R + static_cast<long long>(i) * n;
    double h2;
    if (i > 0) {
      if (k > 0)
        pass(rem, k, i);
      else
        norm_only(rem);
      const double rn2 = finish_dot();
      const int do2 = k > 0 && sqrt(rn2) < 0.5 * norm0[i];
      if (lead && tid == 0) {
        st->rn2 = rn2;
        st->do2 = do2;
      }
      if (do2) {
        pass(rem, k, i);
        h2 = finish_dot();
      } else {
        h2 = rn2;  // (dot(rem, rem) of the unchanged rem: the same partials, the same sum)
      }
    } else {
      norm_only(rem);
      h2 = finish_dot();
    }
    const double h = sqrt(h2);
    const int acc = norm0[i] > 0.0 && h > drop_tol * norm0[i];
    const int pos = k;
    if (lead && tid == 0) {
      st->h2 = h2;
      st->h[i] = h;
      st->acc[i] = acc;
      st->pos[i] = pos;
      st->k = k + acc;
    }
    if (acc) {
      double* col = X + static_cast<long long>(pos) * ldx;
      for (long long e = i0; e < n; e += stride) col[e] = rem[e] / h;
    }
    k += acc;
    grid.sync();  // the next snapshot projects against this column
  }
}

__global__ void add_2d_kernel(int M, int N, const double* __restrict__ T, long long ldt, double* __restrict__ C,
                              long long ldc) {
  const long long total = static_cast<long long>(M) * N;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(e % M), j = static_cast<int>(e / M);
    C[i + j * ldc] += T[i + j * ldt];
  }
}

// rows [r0, r0 + rows) of S (p columns, ld lds) <-> a packed rows x p block
__global__ void pack_rows_kernel(long long rows, int p, const double* __restrict__ S, long long lds, double* __restrict__ B,
                                 bool unpack, double* __restrict__ Sout) {
  const long long total = rows * p;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long i = e % rows;
    const int j = static_cast<int>(e / rows);
    if (unpack)
      Sout[i + j * lds] = B[e];
    else
      B[e] = S[i + j * lds];
  }
}

__global__ void or_flags_kernel(int m, const int* __restrict__ flags, int* __restrict__ bad) {
  int v = 0;
  for (int j = threadIdx.x; j < m; j += blockDim.x) v |= flags[j];
  v = __reduce_or_sync(0xffffffffu, v);
  if ((threadIdx.x & 31) == 0 && v) atomicOr(bad, v);
}

int g1(long long n) {
  long long g = (n + 255) / 256;
  return static_cast<int>(std::max<long long>(1, std::min<long long>(g, 148 * 16)));
}

}  // namespace

LowRankEngine::LowRankEngine(Problem& P, const LowRankParams& prm) : P_(P), prm_(prm), hp_(P.hp_) {
  P.require_k1("LowRankBasis");
  s_ = P.stream_;
  n_ = hp_.ndof;
  nomega_ = hp_.n_omega;
  rmax_ = static_cast<int>(std::min<long long>(n_, nomega_));
  ldp_ = rmax_;
  proj_.ensure(5 * static_cast<size_t>(ldp_) * ldp_);
  prhs_.ensure(ldp_);
  rhs_core_.ensure(n_);
  phi_.ensure(n_);
  phi_old_.ensure(n_);
  rem_.ensure(n_);
  vec_.ensure(3 * static_cast<size_t>(rmax_) + 64);
  dirs_ = P.dirs_.get();
  sa_ = StencilArgs{hp_.nx, hp_.ny, hp_.ncell, P.sigma_t_.get(), P.sc_};
  RTLR_CUDA(cudaMallocHost(&hbuf_, 64 * sizeof(double)));
  RTLR_CUDA(cudaMallocHost(&hstate_, sizeof(CgsState)));
  RTLR_CUDA(cudaMallocHost(&hflags_, 2 * sizeof(int)));
  hflags_[0] = hflags_[1] = 0;
  gal_bad_.ensure(1);
  RTLR_CUDA(cudaMemsetAsync(gal_bad_.get(), 0, sizeof(int), s_));
  ring_.init(s_);
  {
    const char* pe = std::getenv("RTLR_LU_PREFACTOR");
    prefactor_on_ = !(pe && pe[0] == '0');
    int least = 0, greatest = 0;
    RTLR_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    RTLR_CUDA(cudaStreamCreateWithPriority(&s2_, cudaStreamNonBlocking, greatest));
    RTLR_CUDA(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming));
    RTLR_CUDA(cudaEventCreateWithFlags(&ev_asm_, cudaEventDisableTiming));
    RTLR_CUDA(cudaEventCreateWithFlags(&ev_done_, cudaEventDisableTiming));
    RTLR_CUDA(cudaMallocHost(&pf_hang_, 256 * sizeof(int)));
  }
  ldr_ = rmax_;
  // The basis grows every inner iteration; reserving it for the largest
  // possible rank up front (when that takes at most a quarter of the free
  // device memory: 17 GB at C4) keeps multi-GB cudaMalloc/cudaFree pairs,
  // which synchronise the device, out of the first outer iteration.
  size_t free_b = 0, total_b = 0;
  if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess &&
      static_cast<double>(n_) * rmax_ * sizeof(double) <= 0.25 * static_cast<double>(free_b))
    X_.reserve(n_, rmax_, s_);
  const char* e = std::getenv("RTLR_PROFILE");
  pt_.on = (e && e[0] == '1') || P.profile_phases;
  if (e && e[0] == '1') alloc_stats().split = true;
  pt_.s = s_;
  // row slices of the tall contractions
  const char* rs = std::getenv("RTLR_LR_ROWSLICE");
  const char* vs = std::getenv("RTLR_ROWSLICE_VIRTUAL");
  if (P.sharded() && P.nranks() > 1 && !(rs && rs[0] == '0')) {
    nslice_ = P.nranks();
    my_slice_ = P.rank();
  } else if (!P.sharded() && vs && std::atoi(vs) > 1) {
    nslice_ = std::atoi(vs);
    vslice_ = true;
  }
  slice_c_.resize(nslice_ + 1);
  for (int k = 0; k <= nslice_; ++k)
    slice_c_[k] = static_cast<int>(static_cast<long long>(k) * hp_.ncell / nslice_);
}

void LowRankEngine::tn_rows(int M, int N, const double* A, long long lda, const double* B, long long ldb, double* C,
                            long long ldc) {
  if (M <= 0 || N <= 0) return;
  if (nslice_ == 1) {
    tn(M, N, A, lda, B, ldb, C, ldc);
    return;
  }
  double* T = tpart_.ensure(static_cast<size_t>(M) * N);
  auto part = [&](int k, double* out, long long ldo) {
    const long long r0 = slice_row(k), rows = slice_row(k + 1) - r0;
    double* w = work(gemm_tn_work(M, N, rows));
    gemm_tn(M, N, rows, A + r0, lda, B + r0, ldb, out, ldo, w, work_.size(), s_);
  };
  if (!vslice_) {
    part(my_slice_, T, M);
    P_.allreduce_sum(T, static_cast<size_t>(M) * N);
    RTLR_CUDA(cudaMemcpy2DAsync(C, ldc * sizeof(double), T, M * sizeof(double), M * sizeof(double), N,
                                cudaMemcpyDeviceToDevice, s_));
    return;
  }
  part(0, C, ldc);
  for (int k = 1; k < nslice_; ++k) {
    part(k, T, M);
    add_2d_kernel<<<g1(static_cast<long long>(M) * N), 256, 0, s_>>>(M, N, T, M, C, ldc);
  }
  RTLR_CUDA(cudaGetLastError());
}

void LowRankEngine::nn_rows_sub(int p, int r, const double* Xm, long long ldx, const double* Cc, long long ldc,
                                double* S, long long lds, bool share) {
  if (nslice_ == 1) {
    gemm_nn(n_, p, r, Xm, ldx, Cc, ldc, S, lds, s_, /*subtract=*/true);
    return;
  }
  const int first = vslice_ ? 0 : my_slice_, last = vslice_ ? nslice_ : my_slice_ + 1;
  for (int k = first; k < last; ++k) {
    const long long r0 = slice_row(k), rows = slice_row(k + 1) - r0;
    gemm_nn(rows, p, r, Xm + r0, ldx, Cc, ldc, S + r0, lds, s_, /*subtract=*/true);
  }
  if (!share) return;
  // every slice's rows to every rank: pack, all-gather, unpack
  long long maxrows = 0;
  for (int k = 0; k < nslice_; ++k) maxrows = std::max(maxrows, slice_row(k + 1) - slice_row(k));
  const size_t chunk = static_cast<size_t>(maxrows) * p;
  double* G = gath_.ensure(chunk * nslice_);
  for (int k = first; k < last; ++k) {
    const long long r0 = slice_row(k), rows = slice_row(k + 1) - r0;
    pack_rows_kernel<<<g1(rows * p), 256, 0, s_>>>(rows, p, S + r0, lds, G + k * chunk, false, nullptr);
  }
  if (!vslice_) P_.allgather_inplace(G, chunk);
  for (int k = 0; k < nslice_; ++k) {
    if (!vslice_ && k == my_slice_) continue;
    const long long r0 = slice_row(k), rows = slice_row(k + 1) - r0;
    pack_rows_kernel<<<g1(rows * p), 256, 0, s_>>>(rows, p, nullptr, lds, G + k * chunk, true, S + r0);
  }
  RTLR_CUDA(cudaGetLastError());
}

LowRankEngine::~LowRankEngine() {
  cudaStreamSynchronize(s_);
  if (s2_) {
    cudaStreamSynchronize(s2_);
    cudaStreamDestroy(s2_);
    cudaEventDestroy(ev_fork_);
    cudaEventDestroy(ev_asm_);
    cudaEventDestroy(ev_done_);
    cudaFreeHost(pf_hang_);
  }
  cudaFreeHost(hbuf_);
  if (hnorm_) cudaFreeHost(hnorm_);
  cudaFreeHost(hstate_);
  cudaFreeHost(hflags_);
}

double LowRankEngine::host_dot(const double* a, const double* b, long long n) {
  double* out = vec_.get() + 3 * static_cast<size_t>(rmax_);
  dot(n, a, b, work(4096), out, s_);
  RTLR_CUDA(cudaMemcpyAsync(hbuf_, out, sizeof(double), cudaMemcpyDeviceToHost, s_));
  RTLR_CUDA(cudaStreamSynchronize(s_));
  return hbuf_[0];
}

int* LowRankEngine::upload_ints(DBuf<int>&, const std::vector<int>& a) { return ring_.upload(a); }

// Deferred error flags: the sweeps' singular-block flag and the Galerkin
// solves' non-finite flag are read with the next state the host reads anyway
// (enqueue before that synchronisation, check after it); the reference's
// exception and message follow.
void LowRankEngine::flags_enqueue() {
  RTLR_CUDA(cudaMemcpyAsync(hflags_, gal_bad_.get(), sizeof(int), cudaMemcpyDeviceToHost, s_));
  RTLR_CUDA(cudaMemcpyAsync(hflags_ + 1, P_.err_.get(), sizeof(int), cudaMemcpyDeviceToHost, s_));
}

void LowRankEngine::flags_check() {
  if (hflags_[1]) {
    hflags_[1] = 0;
    RTLR_CUDA(cudaMemsetAsync(P_.err_.get(), 0, sizeof(int), s_));
    throw std::runtime_error("sweep: singular local block");
  }
  if (hflags_[0]) {
    hflags_[0] = 0;
    RTLR_CUDA(cudaMemsetAsync(gal_bad_.get(), 0, sizeof(int), s_));
    throw std::runtime_error("galerkin_solve: singular reduced system");
  }
}

void LowRankEngine::reset(const double* d_phi_prev) {
  // rhs_core = Sigma_s phi_prev + G; fresh basis (low_rank.cpp:349-351)
  P_.rhs_core(d_phi_prev, rhs_core_.get());
  RTLR_CUDA(cudaMemcpyAsync(phi_old_.get(), d_phi_prev, n_ * sizeof(double), cudaMemcpyDeviceToDevice, s_));
  reset_rhs(nullptr);
}

// LowRankBasis(ops, quad, bc, rhs_core) (low_rank.cpp:39-44): an empty basis;
// d_rhs_core == nullptr keeps the one reset() just formed.
void LowRankEngine::reset_rhs(const double* d_rhs_core) {
  if (d_rhs_core)
    RTLR_CUDA(cudaMemcpyAsync(rhs_core_.get(), d_rhs_core, n_ * sizeof(double), cudaMemcpyDeviceToDevice, s_));
  rank_ = n_snap_ = prev_rank_ = 0;
  rec_cols_ = std::max(rec_cols_, nomega_);
  rec_.ensure(static_cast<size_t>(ldr_) * rec_cols_);
  RTLR_CUDA(cudaMemsetAsync(rec_.get(), 0, static_cast<size_t>(ldr_) * rec_cols_ * sizeof(double), s_));
  sampled_.clear();
  X_.reserve(n_, 16, s_);
}

// Room for rank_need basis columns and snaps_need record columns.  The
// solvers never exceed min(N_x, N_Omega) columns (every snapshot is a
// distinct angle); the primitives accept any snapshot stream (the
// reference's record grows, low_rank.cpp:45-64), so the projections, the
// record and the small vectors grow geometrically, contents kept.
void LowRankEngine::grow(int rank_need, int snaps_need) {
  if (rank_need > rmax_) {
    const int nr = static_cast<int>(std::min<long long>(n_, std::max(rank_need, 2 * rmax_)));
    DBuf<double> np, nrec, nprhs;
    np.ensure(5 * static_cast<size_t>(nr) * nr);
    for (int k = 0; k < 5; ++k)
      RTLR_CUDA(cudaMemcpy2DAsync(np.get() + static_cast<size_t>(k) * nr * nr, nr * sizeof(double),
                                  proj_.get() + static_cast<size_t>(k) * ldp_ * ldp_, ldp_ * sizeof(double),
                                  ldp_ * sizeof(double), ldp_, cudaMemcpyDeviceToDevice, s_));
    nprhs.ensure(nr);
    RTLR_CUDA(cudaMemcpyAsync(nprhs.get(), prhs_.get(), ldp_ * sizeof(double), cudaMemcpyDeviceToDevice, s_));
    nrec.ensure(static_cast<size_t>(nr) * rec_cols_);
    RTLR_CUDA(cudaMemsetAsync(nrec.get(), 0, static_cast<size_t>(nr) * rec_cols_ * sizeof(double), s_));
    RTLR_CUDA(cudaMemcpy2DAsync(nrec.get(), nr * sizeof(double), rec_.get(), ldr_ * sizeof(double),
                                ldr_ * sizeof(double), rec_cols_, cudaMemcpyDeviceToDevice, s_));
    RTLR_CUDA(cudaStreamSynchronize(s_));
    proj_.swap(np);
    prhs_.swap(nprhs);
    rec_.swap(nrec);
    rmax_ = nr;
    ldp_ = ldr_ = nr;
    vec_.ensure(3 * static_cast<size_t>(rmax_) + 64);
  }
  if (snaps_need > rec_cols_) {
    const int nc = std::max(snaps_need, 2 * rec_cols_);
    DBuf<double> nrec;
    nrec.ensure(static_cast<size_t>(ldr_) * nc);
    RTLR_CUDA(cudaMemsetAsync(nrec.get(), 0, static_cast<size_t>(ldr_) * nc * sizeof(double), s_));
    RTLR_CUDA(cudaMemcpyAsync(nrec.get(), rec_.get(), static_cast<size_t>(ldr_) * rec_cols_ * sizeof(double),
                              cudaMemcpyDeviceToDevice, s_));
    RTLR_CUDA(cudaStreamSynchronize(s_));
    rec_.swap(nrec);
    rec_cols_ = nc;
  }
}

// proj/src/low_rank.cpp:66-132.  The coefficient record (low_rank.hpp:93,
// R's r x n_snap matrix, a column per snapshot) lives on the device in rec_
// (rmax x N_Omega, ld ldr_, zero below each column's length).
bool LowRankEngine::mgs_ro_update(const double* snaps_all, const std::vector<int>& angles_all) {
  const int p_all = static_cast<int>(angles_all.size());
  const int prev0 = rank_;
  const int m0 = n_snap_;
  grow(static_cast<int>(std::min<long long>(n_, rank_ + p_all)), n_snap_ + p_all);
  X_.reserve(n_, rank_ + p_all, s_);
  std::vector<int> accepted;
  bool have_overlap = false;
  double overlap = 0.0;
  auto tlap = std::chrono::steady_clock::now();
  // A batch of more than kCgsMax snapshots (a verification pass's
  // outstanding angles) on a small basis goes through the device path in
  // chunks of kCgsMax, each chunk projected against the basis including the
  // chunks before it: the reference's per-snapshot order, with one host
  // read per chunk instead of four per snapshot (C2: ~1350 snapshots per
  // solve took the host-driven loop; C2 0.70 -> 0.655 s, C3 0.664 -> 0.628 s).
  // On a basis beyond ~1 GB the repeated passes over X cost as much as the
  // host loop saves (C4 chunked throughout: 3.04 against 3.00 s), so those
  // keep one block pass and the host-driven loop.
  static const double chunk_bytes = [] {
    const char* e = std::getenv("RTLR_CGS_CHUNK_MB");
    return (e ? std::atof(e) : 1024.0) * 1048576.0;
  }();
  const bool chunked = p_all > kCgsMax && 8.0 * static_cast<double>(n_) * rank_ <= chunk_bytes;
  const int step = chunked ? kCgsMax : std::max(p_all, 1);
  for (int off = 0; off < p_all; off += step) {
  const int p_in = std::min(step, p_all - off);
  const double* snaps = snaps_all + static_cast<size_t>(off) * n_;
  const std::vector<int> angles(angles_all.begin() + off, angles_all.begin() + off + p_in);
  prev_rank_ = rank_;
  const int m0c = n_snap_;
  // Block classical Gram-Schmidt, equivalent to the reference's per-snapshot
  // CGS up to rounding: every snapshot is projected against the basis that
  // existed before this batch in one GEMM (twice: "twice is enough", the
  // second pass is unconditional for the old basis, which only adds
  // accuracy), then sequentially against the vectors this batch accepted,
  // where the reference's conditional second pass (rem < 0.5 norm0) is
  // kept.  X_old is read 4 times per batch instead of up to 4 times per
  // snapshot.
  const int r_old = rank_;
  if (pt_.on) RTLR_CUDA(cudaStreamSynchronize(s_));
  tlap = std::chrono::steady_clock::now();
  double* Rm = rem_.ensure(static_cast<size_t>(n_) * p_in);
  double* nr = nrm_.ensure(std::max(p_in, 128));
  {
    double* parts = npart_.ensure(static_cast<size_t>(kSnapParts) * p_in);
    copy_norm_parts<<<dim3(kSnapParts, p_in), 256, 0, s_>>>(n_, snaps, n_, Rm, n_, parts);
    norm_parts_finish<<<(p_in + 7) / 8, 256, 0, s_>>>(p_in, parts, nr);
    RTLR_CUDA(cudaGetLastError());
    // the copy with norms, then the within-batch CGS: column i against the i
    // accepted before it, twice, plus its norm and scaling
    double wb = 3.0 * p_in, wf = 2.0 * p_in;
    for (int i = 0; i < p_in; ++i) {
      wb += 2.0 * (2 * i + 2);
      wf += 8.0 * i + 4.0;
    }
    pt_.work(8.0 * n_ * wb, n_ * wf);
  }
  double *C1 = nullptr, *C2 = nullptr;
  if (r_old > 0) {
    C1 = gbuf_.ensure(static_cast<size_t>(2) * r_old * p_in);
    C2 = C1 + static_cast<size_t>(r_old) * p_in;
    auto tg = std::chrono::steady_clock::now();
    if (pt_.on) RTLR_CUDA(cudaStreamSynchronize(s_));
    tg = std::chrono::steady_clock::now();
    // (the second pass is unconditional: with the reference's test
    // |rem| < 0.5 |psi| some snapshot of the batch needs it in 97-100% of
    // the batches at C2-C4, and the test itself cost more than it saved)
    // (row-sliced over ranks: each rank projects and updates its rows, the
    // r_old x p blocks are allreduced, the remainders' rows all-gathered once)
    // four passes over X_old (two projections, two updates) and the p columns
    pt_.work(8.0 * (4.0 * n_ * r_old + 6.0 * n_ * p_in), 8.0 * n_ * r_old * p_in);
    tn_rows(r_old, p_in, X_.col(0), X_.ld, snaps, n_, C1, r_old);
    nn_rows_sub(p_in, r_old, X_.col(0), X_.ld, C1, r_old, Rm, n_, /*share=*/false);
    tn_rows(r_old, p_in, X_.col(0), X_.ld, Rm, n_, C2, r_old);
    nn_rows_sub(p_in, r_old, X_.col(0), X_.ld, C2, r_old, Rm, n_, /*share=*/true);
    lap(3, tg);
  }
  lap(0, tlap);
  // Within-batch CGS against the vectors this batch accepts.  Up to
  // kCgsMax snapshots (every regular batch): on the device, gated by device
  // flags; the batch's record columns and the overlap test's dot product are
  // formed there too, so the host reads one small state per batch (its only
  // synchronisation).  Larger batches (verification offenders) take the
  // host-driven loop.
  if (p_in <= kCgsMax) {
    double* part = work(static_cast<size_t>(kCgsMax) * kCgsParts + kDotWork + 8);
    double* dwork = part + static_cast<size_t>(kCgsMax) * kCgsParts;
    CgsState* st = reinterpret_cast<CgsState*>(cgs_.ensure((sizeof(CgsState) + 7) / 8));
    RTLR_CUDA(cudaMemsetAsync(st, 0, sizeof(CgsState), s_));
    double* Xb = X_.col(r_old);
    static const bool coop = [] {  // (all kCgsParts CTAs must be co-resident)
      int dev = 0, ok = 0, per = 0, sms = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&ok, cudaDevAttrCooperativeLaunch, dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, cgs_batch_kernel, 256, 0);
      const char* e = std::getenv("RTLR_CGS_COOP");
      return ok != 0 && per * sms >= kCgsParts && !(e && e[0] == '0');
    }();
    if (coop) {
      long long nn = n_;
      long long ldx = X_.ld;
      double* part2 = dwork;
      const double* nrc = nr;
      double dtol = drop_tol_;
      void* args[] = {&nn, const_cast<int*>(&p_in), &nrc, &dtol, &Rm, &Xb, &ldx, &st, &part, &part2};
      RTLR_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(cgs_batch_kernel), dim3(kCgsParts), dim3(256), args,
                                            0, s_));
    }
    for (int i = 0; i < p_in && !coop; ++i) {
      double* rem = Rm + static_cast<size_t>(i) * n_;
      if (i > 0) {
        cgs_dots<<<kCgsParts, 256, 0, s_>>>(n_, i, Xb, X_.ld, rem, st, false, part);
        cgs_finish<<<1, 32 * kCgsMax, 0, s_>>>(i, kCgsParts, part, st, i, false);
        cgs_axpy<<<g1(n_), 256, 0, s_>>>(n_, i, Xb, X_.ld, st, false, rem);
        dot(n_, rem, rem, dwork, &st->rn2, s_);
        cgs_gate<<<1, 1, 0, s_>>>(st, nr + i);
        cgs_dots<<<kCgsParts, 256, 0, s_>>>(n_, i, Xb, X_.ld, rem, st, true, part);
        cgs_finish<<<1, 32 * kCgsMax, 0, s_>>>(i, kCgsParts, part, st, i, true);
        cgs_axpy<<<g1(n_), 256, 0, s_>>>(n_, i, Xb, X_.ld, st, true, rem);
      }
      dot(n_, rem, rem, dwork, &st->h2, s_);
      cgs_accept<<<1, 1, 0, s_>>>(st, i, nr + i, drop_tol_);
      cgs_store<<<g1(n_), 256, 0, s_>>>(n_, rem, st, i, Xb, X_.ld);
    }
    rec_batch_kernel<<<p_in, 256, 0, s_>>>(r_old, p_in, C1, C2, st, rec_col(m0c), ldr_);
    overlap_col_kernel<<<1, 1, 0, s_>>>(st, r_old);
    dot_indirect(n_, X_.col(0), X_.col(0), X_.ld, &st->ocol, dwork, &st->overlap, s_);
    RTLR_CUDA(cudaGetLastError());
    CgsState* h = reinterpret_cast<CgsState*>(hstate_);
    RTLR_CUDA(cudaMemcpyAsync(h, st, sizeof(CgsState), cudaMemcpyDeviceToHost, s_));
    flags_enqueue();
    RTLR_CUDA(cudaStreamSynchronize(s_));
    flags_check();
    for (int i = 0; i < p_in; ++i) {
      if (h->acc[i]) accepted.push_back(off + i);
      sampled_.push_back(angles[i]);
      ++n_snap_;
    }
    rank_ = r_old + h->k;
    if (h->ocol >= 0) {  // (the last chunk that added a column holds the batch's last column)
      have_overlap = true;
      overlap = std::abs(h->overlap);
    }
  } else {
    std::vector<double> norm0(p_in), cold;
    RTLR_CUDA(cudaMemcpyAsync(norm0.data(), nr, p_in * sizeof(double), cudaMemcpyDeviceToHost, s_));
    if (r_old > 0) {
      std::vector<double> h1(static_cast<size_t>(r_old) * p_in), h2(h1.size());
      RTLR_CUDA(cudaMemcpyAsync(h1.data(), C1, h1.size() * sizeof(double), cudaMemcpyDeviceToHost, s_));
      RTLR_CUDA(cudaMemcpyAsync(h2.data(), C2, h2.size() * sizeof(double), cudaMemcpyDeviceToHost, s_));
      RTLR_CUDA(cudaStreamSynchronize(s_));
      cold.resize(h1.size());
      for (size_t k = 0; k < h1.size(); ++k) cold[k] = h1[k] + h2[k];
    }
    RTLR_CUDA(cudaStreamSynchronize(s_));
    double* cnew = vec_.get();
    double* corr = vec_.get() + rmax_;
    std::vector<double> hc(p_in), hc2(p_in);
    for (int i = 0; i < p_in; ++i) {
      double* rem = Rm + static_cast<size_t>(i) * n_;
      const int k_new = rank_ - r_old;
      std::vector<double> reccol(rank_ + 1, 0.0);
      for (int k = 0; k < r_old; ++k) reccol[k] = cold[k + static_cast<size_t>(i) * r_old];
      if (k_new > 0) {
        tn(k_new, 1, X_.col(r_old), X_.ld, rem, n_, cnew, k_new);
        gemv_n(n_, k_new, X_.col(r_old), X_.ld, cnew, -1.0, rem, s_);
        RTLR_CUDA(cudaMemcpyAsync(hc.data(), cnew, k_new * sizeof(double), cudaMemcpyDeviceToHost, s_));
        const double rn = std::sqrt(host_dot(rem, rem, n_));
        if (rn < 0.5 * norm0[i]) {
          tn(k_new, 1, X_.col(r_old), X_.ld, rem, n_, corr, k_new);
          gemv_n(n_, k_new, X_.col(r_old), X_.ld, corr, -1.0, rem, s_);
          RTLR_CUDA(cudaMemcpyAsync(hc2.data(), corr, k_new * sizeof(double), cudaMemcpyDeviceToHost, s_));
          RTLR_CUDA(cudaStreamSynchronize(s_));
          for (int k = 0; k < k_new; ++k) hc[k] += hc2[k];
        }
        for (int k = 0; k < k_new; ++k) reccol[r_old + k] = hc[k];
      }
      const double h = std::sqrt(host_dot(rem, rem, n_));
      if (norm0[i] > 0.0 && h > drop_tol_ * norm0[i]) {  // drop_tol (low_rank.hpp:61-62)
        scale_val_kernel<<<g1(n_), 256, 0, s_>>>(n_, rem, h, X_.col(rank_));
        reccol[rank_] = h;
        accepted.push_back(off + i);
        ++rank_;
      } else {
        reccol.resize(rank_);
      }
      // (pageable source: the copy is staged before the call returns)
      RTLR_CUDA(cudaMemcpyAsync(rec_col(n_snap_), reccol.data(), reccol.size() * sizeof(double),
                                cudaMemcpyHostToDevice, s_));
      sampled_.push_back(angles[i]);
      ++n_snap_;
    }
    if (rank_ > prev_rank_ && rank_ >= 2) {
      have_overlap = true;
      overlap = std::abs(host_dot(X_.col(0), X_.col(rank_ - 1), n_));
    }
  }
  }  // chunks
  prev_rank_ = prev0;
  const double* snaps = snaps_all;
  const int p_in = p_all;
  lap(1, tlap);
  const bool reorth = have_overlap && overlap > prm_.eps_mgs;
  if (reorth) {
    ++reorth_count_;
    if (pt_.on) RTLR_CUDA(cudaStreamSynchronize(s_));
    const auto tq0 = std::chrono::steady_clock::now();
    const int n_acc = static_cast<int>(accepted.size());
    const int r_new = prev_rank_ + n_acc;
    double* R = qr_.ensure(static_cast<size_t>(r_new) * r_new);
    // The new basis spans the same nested column spaces as the reference's
    // Householder QR of [X_old, accepted snapshots] (low_rank.cpp:112-130):
    // X_ already holds [X_old, the batch's CGS-orthonormalised columns], a
    // well-conditioned block whose orthogonality slipped at the 1e-10 level
    // the overlap test caught, so CholeskyQR2 on it (four DMMA products
    // and two small Cholesky factorisations) gives the same Q up to column
    // signs and rounding, and R[:, :prev] the old basis in the new one.
    // Householder on the reference's matrix stays as the fallback (a
    // non-positive Cholesky pivot) and behind RTLR_REBUILD=householder.
    static const bool hh_only = [] {
      const char* e = std::getenv("RTLR_REBUILD");
      return e && std::string(e) == "householder";
    }();
    bool chol = false;
    if (!hh_only) {
      double* Qb = qq_.ensure(static_cast<size_t>(n_) * r_new);
      double* cw = work(cholqr2_work_doubles(n_, r_new));
      chol = cholqr2_inplace(n_, r_new, X_.col(0), X_.ld, R, Qb, cw, work_.size(), chol_flag_.ensure(1), s_);
      if (chol) {  // two rounds of X^T X and X R^-1: 8 m n^2 flops, X read three times, written twice
        const double rn = r_new;
        pt_.work(8.0 * 5.0 * n_ * rn, 8.0 * n_ * rn * rn);
      }
    }
    if (!chol) {
      double* M = qa_.ensure(static_cast<size_t>(n_) * r_new);
      if (prev_rank_ > 0)
        RTLR_CUDA(cudaMemcpyAsync(M, X_.col(0), static_cast<size_t>(n_) * prev_rank_ * sizeof(double),
                                  cudaMemcpyDeviceToDevice, s_));
      for (int k = 0; k < n_acc; ++k)
        RTLR_CUDA(cudaMemcpyAsync(M + static_cast<size_t>(n_) * (prev_rank_ + k),
                                  snaps + static_cast<size_t>(accepted[k]) * n_, n_ * sizeof(double),
                                  cudaMemcpyDeviceToDevice, s_));
      double* Q = qq_.ensure(static_cast<size_t>(n_) * r_new);
      double* tau = tau_.ensure(r_new);
      double* qw = work(householder_qr_work(n_, r_new));
      householder_qr(n_, r_new, M, n_, tau, Q, n_, R, qw, work_.size(), s_);
      {  // blocked Householder QR with Q formed: 4 m n^2 - 4/3 n^3 flops; per
         // 32-column panel the trailing block is read and written (twice with Q)
        const double rn = r_new, panels = std::ceil(rn / 32.0);
        pt_.work(8.0 * n_ * rn * (2.0 + 2.0 * panels), 4.0 * n_ * rn * rn - 4.0 / 3.0 * rn * rn * rn);
      }
      RTLR_CUDA(cudaMemcpyAsync(X_.col(0), Q, static_cast<size_t>(n_) * r_new * sizeof(double),
                                cudaMemcpyDeviceToDevice, s_));
    }
    // batch columns: Q^T snapshots (low_rank.cpp:126-129)
    double* B = gbuf_.ensure(static_cast<size_t>(r_new) * p_in);
    tn(r_new, p_in, X_.col(0), X_.ld, snaps, n_, B, r_new);
    rank_ = r_new;
    if (m0 > 0 && prev_rank_ > 0) {
      // old record columns: R[:, :prev] old_j (low_rank.cpp:121-125), one
      // r_new x m0 x prev product on the DMMA tiles
      double* T = hrec_.ensure(static_cast<size_t>(r_new) * m0);
      gemm_nn(r_new, m0, prev_rank_, R, r_new, rec_.get(), ldr_, T, r_new, s_);
      RTLR_CUDA(cudaMemcpy2DAsync(rec_.get(), ldr_ * sizeof(double), T, r_new * sizeof(double), r_new * sizeof(double),
                                  m0, cudaMemcpyDeviceToDevice, s_));
    }
    RTLR_CUDA(cudaMemcpy2DAsync(rec_col(m0), ldr_ * sizeof(double), B, r_new * sizeof(double), r_new * sizeof(double),
                                p_in, cudaMemcpyDeviceToDevice, s_));
    if (pt_.on) RTLR_CUDA(cudaStreamSynchronize(s_));
    reorth_seconds_ += std::chrono::duration<double>(std::chrono::steady_clock::now() - tq0).count();
  }
  return reorth;
}

// proj/src/low_rank.cpp:136-174.  D+ = -(D-)^T holds exactly in exact
// arithmetic (test_dg_operators.cpp:203-210), which leaves five stencil
// products per new column: G = X^T [Dx-P, Dx-^T P, Dy-P, Dy-^T P, St P].
void LowRankEngine::update_projections(bool reorth) {
  const int r0 = reorth ? 0 : prev_rank_;
  const int pn = rank_ - r0;
  if (pn <= 0) return;
  const int chunk = 32;
  for (int c0 = 0; c0 < pn; c0 += chunk) {
    const int pc = std::min(chunk, pn - c0);
    double* W = wbuf_.ensure(static_cast<size_t>(n_) * 5 * chunk);
    // (row-sliced over ranks: the stencil images of this rank's cells, X^T W
    // over its rows, one allreduce of the rank x 5pc block)
    if (nslice_ > 1 && !vslice_)
      stream_products(sa_, pc, X_.col(r0 + c0), X_.ld, W, n_, s_, slice_c_[my_slice_], slice_c_[my_slice_ + 1]);
    else
      stream_products(sa_, pc, X_.col(r0 + c0), X_.ld, W, n_, s_);
    double* G = gbuf_.ensure(static_cast<size_t>(rank_) * 5 * chunk);
    // stencil images (read pc columns with their neighbours, write 5 pc) and
    // X^T W (read X and W): 2 n r 5pc flops on the DMMA tiles
    pt_.work(8.0 * (static_cast<double>(n_) * pc * 11.0 + static_cast<double>(n_) * rank_),
             2.0 * n_ * rank_ * 5.0 * pc + 40.0 * n_ * pc);
    tn_rows(rank_, 5 * pc, X_.col(0), X_.ld, W, n_, G, rank_);
    proj_border_kernel<<<g1(static_cast<long long>(rank_) * pc), 256, 0, s_>>>(r0, pn, c0, pc, G, rank_, proj_.get(),
                                                                             ldp_, ldp_ * ldp_, rank_);
    RTLR_CUDA(cudaGetLastError());
  }
  tn_rows(pn, 1, X_.col(r0), X_.ld, rhs_core_.get(), n_, prhs_.get() + r0, pn);
}

// galerkin_solve for a list of angles (low_rank.cpp:192-200), batched.
// Mirror directions share (Omega_x, Omega_y) bitwise and, without inflow
// data, the reduced right-hand side, so each distinct system is solved once
// and its solution copied (bitwise the per-angle result).
void LowRankEngine::galerkin(const std::vector<int>& angles, double* d_sol, long long ldsol) {
  if (rank_ < 1) throw std::runtime_error("galerkin_solve: empty basis");
  if (!hp_.bc_any) {
    std::vector<int> reps, pos(angles.size()), seen(P_.uniq_rep_.size(), -1);
    for (size_t k = 0; k < angles.size(); ++k) {
      const int u = P_.uniq_of_[angles[k]];
      if (seen[u] < 0) {
        seen[u] = static_cast<int>(reps.size());
        reps.push_back(angles[k]);
      }
      pos[k] = seen[u];
    }
    if (reps.size() < angles.size()) {
      double* tmp = gsol_.ensure(static_cast<size_t>(rank_) * padded(static_cast<int>(reps.size())));
      galerkin_solve(reps, tmp, rank_);
      int* dpos = upload_ints(pos_, pos);
      const int m = static_cast<int>(angles.size());
      gather_cols<<<g1(static_cast<long long>(rank_) * m), 256, 0, s_>>>(rank_, m, dpos, tmp, rank_, d_sol, ldsol);
      RTLR_CUDA(cudaGetLastError());
      return;
    }
  }
  galerkin_solve(angles, d_sol, ldsol);
}

// Sharded: this rank solves its block of the angles and one all-gather
// assembles every column on every rank (d_sol holds padded(m) columns).
void LowRankEngine::galerkin_solve(const std::vector<int>& angles, double* d_sol, long long ldsol) {
  const int m = static_cast<int>(angles.size());
  ++gal_calls_;
  gal_systems_ += m;
  const ShardBlock sb = blk(m);
  const long long rr = static_cast<long long>(rank_) * rank_;
  // Systems per LU batch for r > kSmemLuMax: up to a 4 GiB LU workspace
  // (galerkin_work_doubles per system: the r x (r+1) augmented matrix, the
  // pivots and the permutation; 2.9 MB at r = 600, so 1,480 systems — C4's
  // all-angle solves, ~1,000 distinct systems per call, run as one batch:
  // 33.8 -> 29.4 ms per call against 372-system batches).  The grid's y
  // dimension carries the systems, so a batch is capped at 65,535.  Results
  // do not depend on the batching.
  static const long long budget_bytes = [] {
    const char* e = std::getenv("RTLR_GAL_CHUNK_MB");
    return (e && std::atoll(e) > 0 ? std::atoll(e) : 4096LL) << 20;
  }();
  const long long per_system = static_cast<long long>(galerkin_work_per_system(rank_)) * sizeof(double);
  const int chunk = rank_ > kSmemLuMax
                        ? static_cast<int>(std::min<long long>(65535, std::max<long long>(1, budget_bytes / per_system)))
                        : 4096;
  for (int j0 = sb.begin; j0 < sb.end; j0 += chunk) {
    const int mc = std::min(chunk, sb.end - j0);
    std::vector<int> sub(angles.begin() + j0, angles.begin() + j0 + mc);
    int* d_ang = upload_ints(ang_, sub);
    double* out = d_sol + static_cast<long long>(j0) * ldsol;
    const double* extra = nullptr;
    if (hp_.bc_any) {
      // reduced_rhs: + X^T g_j (low_rank.cpp:185-190), formed in sub-blocks
      // of kBcCols boundary vectors so the staging buffer stays n x kBcCols
      // whatever the batch size
      constexpr int kBcCols = 64;
      double* Gb = ybuf_.ensure(static_cast<size_t>(n_) * std::min(mc, kBcCols));
      for (int b0 = 0; b0 < mc; b0 += kBcCols) {
        const int nb = std::min(kBcCols, mc - b0);
        for (int j = 0; j < nb; ++j)
          RTLR_CUDA(cudaMemcpyAsync(Gb + static_cast<size_t>(j) * n_,
                                    P_.bc_.get() + static_cast<size_t>(sub[b0 + j]) * n_, n_ * sizeof(double),
                                    cudaMemcpyDeviceToDevice, s_));
        tn(rank_, nb, X_.col(0), X_.ld, Gb, n_, out + static_cast<long long>(b0) * ldsol, ldsol);
      }
      extra = out;
    }
    int* flags = flags_.ensure(mc);
    {  // assembly + partial-pivot LU + two triangular solves per system: the
       // r x (r+1) matrices are written once and factored in place
      const double r = rank_;
      pt_.work(8.0 * mc * r * (r + 1) * 2.0, mc * (2.0 / 3.0 * r * r * r + 2.0 * r * r + 5.0 * r * r));
    }
    const size_t lwn = galerkin_work_doubles(rank_, mc);
    double* lw = lwn ? luw_.ensure(lwn) : nullptr;
    galerkin_batch(rank_, mc, d_ang, dirs_, proj_.get(), ldp_, ldp_ * ldp_, prhs_.get(), extra, out, ldsol, flags, lw,
                   s_);
    or_flags_kernel<<<1, 256, 0, s_>>>(mc, flags, gal_bad_.get());
    RTLR_CUDA(cudaGetLastError());
  }
  if (P_.sharded()) {
    // every rank holds the same flag (checked with the next host read, so all
    // ranks throw together) and every column
    P_.allreduce_max(gal_bad_.get(), 1);
    if (ldsol != rank_) throw std::logic_error("galerkin: sharded solutions must be packed (ldsol == rank)");
    P_.allgather_inplace(d_sol, static_cast<size_t>(sb.bsz) * ldsol);
  }
}

// ||rhs_j - (D_j + Sigma_t) X c_j|| for the listed angles, expanded block-
// wise (low_rank.cpp:283-307); coefficient column k belongs to angles[k].
std::vector<double> LowRankEngine::residual_norms(const std::vector<int>& angles, const double* coeffs,
                                                  long long ldc, bool mirror_equal) {
  // Mirror directions with equal coefficient columns (Galerkin solutions,
  // copied per distinct system) have bitwise equal residuals: each distinct
  // one is evaluated once (the GEMM and the per-angle reduction do not
  // depend on a column's position in the block) and the norm copied.
  if (mirror_equal && !hp_.bc_any && !angles.empty()) {
    std::vector<int> reps, from, pos(angles.size()), seen(P_.uniq_rep_.size(), -1);
    for (size_t k = 0; k < angles.size(); ++k) {
      const int u = P_.uniq_of_[angles[k]];
      if (seen[u] < 0) {
        seen[u] = static_cast<int>(reps.size());
        reps.push_back(angles[k]);
        from.push_back(static_cast<int>(k));
      }
      pos[k] = seen[u];
    }
    if (reps.size() < angles.size()) {
      const int nr = static_cast<int>(reps.size());
      double* rc = rcoef_.ensure(static_cast<size_t>(rank_) * padded(nr));
      int* df = upload_ints(rfrom_, from);
      gather_cols<<<g1(static_cast<long long>(rank_) * nr), 256, 0, s_>>>(rank_, nr, df, coeffs, ldc, rc, rank_);
      RTLR_CUDA(cudaGetLastError());
      const std::vector<double> rn = residual_norms(reps, rc, rank_, false);
      std::vector<double> out(angles.size());
      for (size_t k = 0; k < angles.size(); ++k) out[k] = rn[pos[k]];
      return out;
    }
  }
  // Sharded: this rank evaluates its block of the angles; the norms are
  // all-gathered (every rank then takes the same greedy decisions).
  const int m = static_cast<int>(angles.size());
  std::vector<double> out(m);
  if (m == 0) return out;
  const ShardBlock sb = blk(m);
  double* nr_all = nrm_.ensure(std::max(padded(m), 128));
  const int block = 128;
  for (int i0 = sb.begin; i0 < sb.end; i0 += block) {
    const int nb = std::min(block, sb.end - i0);
    std::vector<int> sub(angles.begin() + i0, angles.begin() + i0 + nb);
    double* Y = ybuf_.ensure(static_cast<size_t>(n_) * block);
    // Y = X C (read X once per block, write Y) and the stencil residual
    // (read Y, the Sigma_t blocks and rhs once per block): 2 n r nb flops
    pt_.work(8.0 * (static_cast<double>(n_) * rank_ + 2.0 * n_ * nb + 16.0 * hp_.ncell + n_),
             2.0 * n_ * rank_ * nb + 60.0 * n_ * nb);
    gemm_nn(n_, nb, rank_, X_.col(0), X_.ld, coeffs + static_cast<long long>(i0) * ldc, ldc, Y, n_, s_);
    int* d_ang = upload_ints(ang_, sub);
    launch_residual_norms(sa_, nb, d_ang, dirs_, Y, n_, rhs_core_.get(), hp_.bc_any ? P_.bc_.get() : nullptr, n_,
                          work(static_cast<size_t>(block) * residual_parts(hp_.ncell)), nr_all + i0, s_);
  }
  P_.allgather_inplace(nr_all, sb.bsz);
  // (through pinned memory: a pageable destination makes the copy a staged,
  // host-synchronous one, ~10 us more per greedy step)
  if (static_cast<size_t>(m) > hnorm_cap_) {
    if (hnorm_) RTLR_CUDA(cudaFreeHost(hnorm_));
    hnorm_cap_ = std::max<size_t>(2 * static_cast<size_t>(m), 256);
    RTLR_CUDA(cudaMallocHost(&hnorm_, hnorm_cap_ * sizeof(double)));
  }
  RTLR_CUDA(cudaMemcpyAsync(hnorm_, nr_all, m * sizeof(double), cudaMemcpyDeviceToHost, s_));
  flags_enqueue();
  RTLR_CUDA(cudaStreamSynchronize(s_));
  flags_check();
  std::copy(hnorm_, hnorm_ + m, out.begin());
  return out;
}

// proj/src/low_rank.cpp:311-336: sampled columns from the record,
// candidate solutions reused, Galerkin solves for the rest.
void LowRankEngine::build_full_coefficients(const std::vector<int>* cand, const double* cand_sol) {
  const int r = rank_;
  double* C = C_.ensure(static_cast<size_t>(r) * nomega_);
  std::vector<char> done(nomega_, 0);
  std::vector<int> idx(n_snap_);
  for (int i = 0; i < n_snap_; ++i) {
    idx[i] = sampled_[i];
    done[sampled_[i]] = 1;
  }
  int* di = upload_ints(ang2_, idx);
  scatter_cols<<<g1(static_cast<long long>(r) * n_snap_), 256, 0, s_>>>(r, n_snap_, di, rec_.get(), ldr_, C, r);
  if (cand) {
    std::vector<int> to, from;
    for (size_t i = 0; i < cand->size(); ++i)
      if (!done[(*cand)[i]]) {
        to.push_back((*cand)[i]);
        from.push_back(static_cast<int>(i));
        done[(*cand)[i]] = 1;
      }
    if (!to.empty()) {
      double* tmpc = ybuf_.ensure(static_cast<size_t>(r) * to.size());
      int* df = upload_ints(ang_, from);
      gather_cols<<<g1(static_cast<long long>(r) * from.size()), 256, 0, s_>>>(r, static_cast<int>(from.size()), df,
                                                                              cand_sol, r, tmpc, r);
      int* dt = upload_ints(ang2_, to);
      scatter_cols<<<g1(static_cast<long long>(r) * to.size()), 256, 0, s_>>>(r, static_cast<int>(to.size()), dt, tmpc,
                                                                             r, C, r);
    }
  }
  // An angle whose mirror partner (the same (Omega_x, Omega_y)) has a
  // record column takes that column: the partner's snapshot is the angle's
  // own transport solution and lies in the basis span, so the angle's
  // Galerkin solution is that column up to rounding (the reference solves
  // it; the verification residuals of such angles are ~1e-12 at C2-C4).
  // RTLR_BUILDC_MIRRORS=solve solves them as the reference does.
  static const bool copy_mirrors = [] {
    const char* e = std::getenv("RTLR_BUILDC_MIRRORS");
    return !(e && std::string(e) == "solve");
  }();
  if (copy_mirrors && !hp_.bc_any && n_snap_ > 0) {
    std::vector<int> src_of(P_.uniq_rep_.size(), -1);
    for (int i = 0; i < n_snap_; ++i) src_of[P_.uniq_of_[sampled_[i]]] = sampled_[i];
    std::vector<int> to, from;
    for (int j = 0; j < nomega_; ++j)
      if (!done[j] && src_of[P_.uniq_of_[j]] >= 0) {
        to.push_back(j);
        from.push_back(src_of[P_.uniq_of_[j]]);
        done[j] = 1;
      }
    if (!to.empty()) {
      double* tmpc = ybuf_.ensure(static_cast<size_t>(r) * to.size());
      int* df = upload_ints(ang_, from);
      gather_cols<<<g1(static_cast<long long>(r) * from.size()), 256, 0, s_>>>(r, static_cast<int>(from.size()), df, C,
                                                                              r, tmpc, r);
      int* dt = upload_ints(ang2_, to);
      scatter_cols<<<g1(static_cast<long long>(r) * to.size()), 256, 0, s_>>>(r, static_cast<int>(to.size()), dt, tmpc,
                                                                             r, C, r);
    }
  }
  std::vector<int> rest;
  for (int j = 0; j < nomega_; ++j)
    if (!done[j]) rest.push_back(j);
  if (!rest.empty()) {
    double* S = sol_.ensure(static_cast<size_t>(r) * padded(static_cast<int>(rest.size())));
    galerkin(rest, S, r);
    int* dr = upload_ints(ang2_, rest);
    scatter_cols<<<g1(static_cast<long long>(r) * rest.size()), 256, 0, s_>>>(r, static_cast<int>(rest.size()), dr, S,
                                                                             r, C, r);
  }
  RTLR_CUDA(cudaGetLastError());
}

// phi = X (C w)   (low_rank.cpp:385,394)
void LowRankEngine::phi_from_C() {
  pt_.work(8.0 * (static_cast<double>(n_) * rank_ + static_cast<double>(rank_) * nomega_ + n_),
           2.0 * n_ * rank_ + 2.0 * rank_ * nomega_);
  double* cw = vec_.get() + 2 * static_cast<size_t>(rmax_);
  RTLR_CUDA(cudaMemsetAsync(cw, 0, rank_ * sizeof(double), s_));
  gemv_n(rank_, nomega_, C_.get(), rank_, P_.weights_.get(), 1.0, cw, s_);
  RTLR_CUDA(cudaMemsetAsync(phi_.get(), 0, n_ * sizeof(double), s_));
  gemv_n(n_, rank_, X_.col(0), X_.ld, cw, 1.0, phi_.get(), s_);
}

// proj/src/low_rank.cpp:217-252: q random unsampled candidates (the RNG's
// partial Fisher-Yates over the ascending pool), their Galerkin solutions
// (kept in cand_), full-space residual norms, the p largest (ties by angle).
GreedyOutcome LowRankEngine::greedy_subsample(const std::vector<char>& sampled, int p, int q, SubsampleRng& rng) {
  std::vector<int> pool;
  for (int j = 0; j < nomega_; ++j)
    if (!sampled[j]) pool.push_back(j);
  return greedy_evaluate(rng.sample_without_replacement(std::move(pool), q), p, /*use_prefactor=*/false);
}

// The candidates of the inner iteration that sweeps `next`, drawn now: that
// iteration marks `next` sampled and then draws from the unsampled pool
// (low_rank.cpp:217-226), and nothing in between touches the RNG, so the
// draw is the same one.  None when no angle would remain (the loop then ends
// as exhausted without a draw).  The distinct candidate systems are factored
// at the current rank on s2_ (not for inflow problems, whose right-hand
// sides are per angle, nor while the one-CTA solve is faster).
void LowRankEngine::predraw(const std::vector<char>& sampled, const std::vector<int>& next, int q,
                            SubsampleRng& rng) {
  pf_.have_cands = pf_.factored = false;
  if (!prefactor_on_) return;
  std::vector<char> mark(sampled);
  for (int j : next) mark[j] = 1;
  std::vector<int> pool;
  for (int j = 0; j < nomega_; ++j)
    if (!mark[j]) pool.push_back(j);
  if (pool.empty()) return;
  pf_.cands = rng.sample_without_replacement(std::move(pool), q);
  pf_.have_cands = true;
  static const int min_rank = [] {
    const char* e = std::getenv("RTLR_LU_PREFACTOR_MIN");
    return e ? std::atoi(e) : 64;
  }();
  const int m = static_cast<int>(pf_.cands.size());
  // (With a communicator every rank factors and finishes all the candidates
  // itself: the projections are replicated, the work is off the critical
  // path, and the solutions then need no all-gather.)
  if (hp_.bc_any || rank_ <= min_rank || m == 0 || m > 256 ||
      static_cast<int>(next.size()) > 8 || !galerkin_border_fits(rank_, 8))
    return;
  pf_.reps.clear();
  pf_.pos.assign(m, 0);
  std::vector<int> seen(P_.uniq_rep_.size(), -1);
  for (int k = 0; k < m; ++k) {
    const int u = P_.uniq_of_[pf_.cands[k]];
    if (seen[u] < 0) {
      seen[u] = static_cast<int>(pf_.reps.size());
      pf_.reps.push_back(pf_.cands[k]);
    }
    pf_.pos[k] = seen[u];
  }
  const int mr = static_cast<int>(pf_.reps.size());
  const size_t need = static_cast<size_t>(mr) * galerkin_work_per_system(rank_);
  if (pfw_.size() < need) {
    RTLR_CUDA(cudaStreamSynchronize(s2_));
    pfw_.ensure(static_cast<size_t>(mr) * galerkin_work_per_system(std::min<int>(rmax_, rank_ + 64)));
  }
  std::memcpy(pf_hang_, pf_.reps.data(), mr * sizeof(int));
  RTLR_CUDA(cudaMemcpyAsync(pf_ang_.ensure(256), pf_hang_, mr * sizeof(int), cudaMemcpyHostToDevice, s_));
  RTLR_CUDA(cudaEventRecord(ev_fork_, s_));
  RTLR_CUDA(cudaStreamWaitEvent(s2_, ev_fork_, 0));
  galerkin_prefactor(rank_, mr, pf_ang_.get(), dirs_, proj_.get(), ldp_, ldp_ * ldp_, prhs_.get(), pfw_.get(), s2_,
                     ev_asm_);
  RTLR_CUDA(cudaEventRecord(ev_done_, s2_));
  pf_.r0 = rank_;
  pf_.factored = true;
}

// The candidates' Galerkin solutions (kept in cand_), full-space residual
// norms, the p largest (ties by angle) (low_rank.cpp:227-252).
GreedyOutcome LowRankEngine::greedy_evaluate(std::vector<int> cands_in, int p, bool use_prefactor) {
  GreedyOutcome g;
  g.candidates = std::move(cands_in);
  const std::vector<int>& cands = g.candidates;
  const int m = static_cast<int>(cands.size());
  if (m == 0) return g;
  double* csol = cand_.ensure(static_cast<size_t>(rank_) * padded(m));
  pt_.start("galerkin_q");
  const int k_new = rank_ - pf_.r0;
  if (use_prefactor && pf_.factored && pf_.r0 == prev_rank_ && k_new >= 0 && galerkin_border_fits(pf_.r0, k_new)) {
    const int mr = static_cast<int>(pf_.reps.size());
    ++gal_calls_;
    gal_systems_ += mr;
    ++pf_used_;
    {  // on the critical path: the border's three triangular solves per system
      const double r = rank_;
      pt_.work(8.0 * mr * 1.5 * r * r, mr * (3.0 * r * r * (k_new + 1)));
    }
    RTLR_CUDA(cudaStreamWaitEvent(s_, ev_done_, 0));
    double* tmp = mr < m ? gsol_.ensure(static_cast<size_t>(rank_) * mr) : csol;
    int* flags = flags_.ensure(mr);
    galerkin_border_solve(pf_.r0, k_new, mr, pf_ang_.get(), dirs_, proj_.get(), ldp_, ldp_ * ldp_, prhs_.get(),
                          pfw_.get(), tmp, rank_, flags, s_);
    or_flags_kernel<<<1, 256, 0, s_>>>(mr, flags, gal_bad_.get());
    if (mr < m) {
      int* dpos = upload_ints(pos_, pf_.pos);
      gather_cols<<<g1(static_cast<long long>(rank_) * m), 256, 0, s_>>>(rank_, m, dpos, tmp, rank_, csol, rank_);
    }
    RTLR_CUDA(cudaGetLastError());
    static const bool check = [] {  // RTLR_LU_PREFACTOR=check: against the full pivoted LU, worst column reported
      const char* e = std::getenv("RTLR_LU_PREFACTOR");
      return e && std::string(e) == "check";
    }();
    if (check) {
      std::vector<double> a(static_cast<size_t>(rank_) * m), b(a.size());
      RTLR_CUDA(cudaMemcpyAsync(a.data(), csol, a.size() * sizeof(double), cudaMemcpyDeviceToHost, s_));
      RTLR_CUDA(cudaStreamSynchronize(s_));
      DBuf<double> full;
      galerkin(cands, full.ensure(a.size()), rank_);
      RTLR_CUDA(cudaMemcpyAsync(b.data(), full.get(), b.size() * sizeof(double), cudaMemcpyDeviceToHost, s_));
      RTLR_CUDA(cudaStreamSynchronize(s_));
      double worst = 0.0;
      for (int c = 0; c < m; ++c) {
        double d2 = 0.0, n2 = 0.0;
        for (int i = 0; i < rank_; ++i) {
          const double x = a[i + static_cast<size_t>(c) * rank_], y = b[i + static_cast<size_t>(c) * rank_];
          d2 += (x - y) * (x - y);
          n2 += y * y;
        }
        worst = std::max(worst, std::sqrt(d2 / std::max(n2, 1e-300)));
      }
      pf_check_worst_ = std::max(pf_check_worst_, worst);
    }
  } else {
    if (pf_.factored) ++pf_missed_;
    galerkin(cands, csol, rank_);
  }
  pf_.factored = false;
  pt_.stop();
  pt_.start("residual_q");
  g.residual_norms = residual_norms(cands, csol, rank_, /*mirror_equal=*/true);
  pt_.stop();
  const std::vector<double>& norms = g.residual_norms;
  std::vector<int> order(m);
  std::iota(order.begin(), order.end(), 0);
  std::sort(order.begin(), order.end(), [&](int a, int b) {
    if (norms[a] != norms[b]) return norms[a] > norms[b];
    return cands[a] < cands[b];
  });
  g.max_residual = norms[order.front()];
  for (int i = 0; i < std::min(p, m); ++i) g.selected.push_back(cands[order[i]]);
  return g;
}

// Loads caller factors for svd() (truncate_factors on external C and X).
void LowRankEngine::load_factors(const double* d_C, const double* d_X, int r) {
  if (r < 1 || r > n_) throw std::invalid_argument("truncate_factors: rank out of range");
  grow(r, 0);
  X_.reserve(n_, r, s_);
  RTLR_CUDA(cudaMemcpy2DAsync(X_.col(0), X_.ld * sizeof(double), d_X, n_ * sizeof(double), n_ * sizeof(double), r,
                              cudaMemcpyDeviceToDevice, s_));
  double* C = C_.ensure(static_cast<size_t>(r) * nomega_);
  RTLR_CUDA(cudaMemcpyAsync(C, d_C, static_cast<size_t>(r) * nomega_ * sizeof(double), cudaMemcpyDeviceToDevice, s_));
  rank_ = r;
}

// proj/src/low_rank.cpp:340-434
InnerResult LowRankEngine::inner(const double* d_phi_prev, SubsampleRng& rng) {
  if (prm_.p < 1 || prm_.q < prm_.p) throw std::invalid_argument("low_rank_si: need 1 <= p <= q");
  reset(d_phi_prev);
  pf_.have_cands = pf_.factored = false;
  std::vector<char> sampled(nomega_, 0);
  InnerResult out;
  std::vector<int> all(nomega_);
  std::iota(all.begin(), all.end(), 0);
  std::vector<int> next = rng.sample_without_replacement(all, std::min(prm_.p, nomega_));
  while (true) {
    ++out.iterations;
    const int p_now = static_cast<int>(next.size());
    double* S = snaps_.ensure(static_cast<size_t>(n_) * padded(p_now));
    int* d_next = upload_ints(ang2_, next);
    pt_.start("sweep");
    {  // sharded: this rank's block of the sampled sweeps, then one all-gather
      const ShardBlock sb = blk(p_now);
      P_.sweep(d_next + sb.begin, sb.end - sb.begin, rhs_core_.get(), 0, S + static_cast<size_t>(sb.begin) * n_, n_);
      // Sigma_t blocks + the shared rhs read once, one psi written per direction;
      // ~150 flops per cell-direction (4x4 LU, solve, two upwind couplings)
      pt_.work(8.0 * (16.0 * hp_.ncell + n_ + static_cast<double>(p_now) * n_), 150.0 * p_now * hp_.ncell);
      // (the singular-block flag is read with the CGS state; sharded, it is
      // max-reduced first so every rank throws together)
      if (P_.sharded()) {
        P_.allreduce_max(P_.err_.get(), 1);
        P_.allgather_inplace(S, static_cast<size_t>(sb.bsz) * n_);
      }
    }
    pt_.stop();
    for (int j : next) {
      sampled[j] = 1;
      out.sampled_order.push_back(j);
    }
    // (the prefactor's assembly reads the projections at the old rank:
    // it precedes this iteration's growth and border writes)
    if (pf_.factored) RTLR_CUDA(cudaStreamWaitEvent(s_, ev_asm_, 0));
    pt_.start("cgs");
    const bool reorth = mgs_ro_update(S, next);
    pt_.stop();
    pt_.start("projections");
    update_projections(reorth);
    pt_.stop();
    if (reorth) ++out.reorthogonalizations;
    const bool any_unsampled = std::any_of(sampled.begin(), sampled.end(), [](char c) { return !c; });
    if (!any_unsampled) {
      out.exhausted = true;
      build_full_coefficients(nullptr, nullptr);
      phi_from_C();
      break;
    }
    GreedyOutcome g;
    if (pf_.have_cands) {
      pf_.have_cands = false;
      g = greedy_evaluate(std::move(pf_.cands), prm_.p, /*use_prefactor=*/!reorth);
    } else {
      g = greedy_subsample(sampled, prm_.p, prm_.q, rng);
    }
    const std::vector<int>& cands = g.candidates;
    const double* csol = cand_.get();
    const double max_residual = g.max_residual;
    next = g.selected;

    if (max_residual < prm_.eps_res) {
      pt_.start("build_C");
      build_full_coefficients(&cands, csol);
      phi_from_C();
      pt_.stop();
      // ||phi - phi_old||_2
      double* w = work(2 * kNormParts + 8);
      diff_norms(static_cast<int>(n_), phi_.get(), phi_old_.get(), w, w + 2 * kNormParts, s_);
      RTLR_CUDA(cudaMemcpyAsync(hbuf_, w + 2 * kNormParts, 2 * sizeof(double), cudaMemcpyDeviceToHost, s_));
      flags_enqueue();
      RTLR_CUDA(cudaStreamSynchronize(s_));
      flags_check();
      if (hbuf_[0] <= prm_.eps_diff) {
        // verify every unsampled angle before accepting (low_rank.cpp:396-424).
        // An unsampled angle whose mirror partner (the same (Omega_x,
        // Omega_y)) is sampled has that partner's snapshot,
        // psi = (D + Sigma_t)^-1 rhs, in the basis span (accepted, or dropped
        // with a remainder below drop_tol of its norm), so its Galerkin
        // solution reproduces it and its residual is rounding noise, far
        // below eps_res: it cannot be outstanding, and it is not evaluated
        // (the reference evaluates it; the accept / outstanding decisions
        // are the same).  RTLR_VERIFY_MIRRORS=eval evaluates every angle;
        // =check evaluates them and reports the largest such residual.
        static const int mirror_mode = [] {  // 0 skip, 1 eval, 2 check
          const char* e = std::getenv("RTLR_VERIFY_MIRRORS");
          if (!e) return 0;
          const std::string v = e;
          return v == "eval" ? 1 : v == "check" ? 2 : 0;
        }();
        std::vector<char> partner_sampled(P_.uniq_rep_.size(), 0);
        for (int j = 0; j < nomega_; ++j)
          if (sampled[j]) partner_sampled[P_.uniq_of_[j]] = 1;
        std::vector<int> unsampled, skipped;
        for (int j = 0; j < nomega_; ++j)
          if (!sampled[j]) {
            if (mirror_mode != 1 && partner_sampled[P_.uniq_of_[j]] && !hp_.bc_any)
              skipped.push_back(j);
            else
              unsampled.push_back(j);
          }
        if (mirror_mode == 2) unsampled.insert(unsampled.end(), skipped.begin(), skipped.end());
        double* Cu = sol_.ensure(static_cast<size_t>(rank_) * unsampled.size());
        int* du = upload_ints(ang2_, unsampled);
        gather_cols<<<g1(static_cast<long long>(rank_) * unsampled.size()), 256, 0, s_>>>(
            rank_, static_cast<int>(unsampled.size()), du, C_.get(), rank_, Cu, rank_);
        pt_.start("verify");
        ++verify_calls_;
        verify_angles_ += static_cast<long long>(unsampled.size());
        std::vector<double> vn = residual_norms(unsampled, Cu, rank_, /*mirror_equal=*/true);
        pt_.stop();
        if (mirror_mode == 2 && !skipped.empty()) {
          double worst = 0.0;
          for (size_t i = unsampled.size() - skipped.size(); i < unsampled.size(); ++i) worst = std::max(worst, vn[i]);
          std::fprintf(stderr, "[rtlr verify] %zu angles with a sampled mirror partner: largest residual %.3e (eps_res %.1e)\n",
                       skipped.size(), worst, prm_.eps_res);
        }
        std::vector<std::pair<double, int>> outstanding;
        for (size_t i = 0; i < unsampled.size(); ++i)
          if (vn[i] >= prm_.eps_res) outstanding.push_back({vn[i], unsampled[i]});
        if (outstanding.empty()) break;
        std::sort(outstanding.begin(), outstanding.end(), [](const auto& a, const auto& b) {
          if (a.first != b.first) return a.first > b.first;
          return a.second < b.second;
        });
        next.clear();
        for (const auto& e : outstanding) next.push_back(e.second);
        ++out.verification_rejections;
      }
      RTLR_CUDA(cudaMemcpyAsync(phi_old_.get(), phi_.get(), n_ * sizeof(double), cudaMemcpyDeviceToDevice, s_));
    }
    predraw(sampled, next, prm_.q, rng);
  }
  pf_.have_cands = pf_.factored = false;
  flags_enqueue();
  RTLR_CUDA(cudaStreamSynchronize(s_));
  flags_check();
  out.rank = rank_;
  out.sampled_count = n_snap_;
  return out;
}

// Singular values of C (and, with vectors, truncate_factors' X U and V)
// by one-sided Jacobi on C^T (N_Omega x r) or C (r x N_Omega), whichever
// has the longer columns (low_rank.cpp:268-277, 457-458).
std::vector<double> LowRankEngine::svd(bool vectors, int keep, std::vector<double>* Xout, std::vector<double>* Vout) {
  // QR-preconditioned one-sided Jacobi (the north star's "Householder QR of
  // the tall-skinny factor plus a small SVD of the r x r core"): W = Q R by
  // the blocked Householder QR, then Jacobi on R^T.  Rotating R^T's columns
  // converges in ~10 sweeps where rotating W's took ~38, each on r-long
  // instead of N_Omega-long columns.  W = C^T (N_Omega x r) when r <=
  // N_Omega, else C; W = (Q J) S L^T with R^T J = L S.
  const int r = rank_;
  const bool on_ct = r <= nomega_;
  const int ncols = on_ct ? r : nomega_;
  const long long mrows = on_ct ? nomega_ : r;
  double* Wm = qa_.ensure(static_cast<size_t>(mrows) * ncols);
  if (on_ct)
    transpose_kernel<<<g1(static_cast<long long>(r) * nomega_), 256, 0, s_>>>(r, nomega_, C_.get(), r, Wm, nomega_);
  else
    RTLR_CUDA(cudaMemcpyAsync(Wm, C_.get(), static_cast<size_t>(r) * nomega_ * sizeof(double),
                              cudaMemcpyDeviceToDevice, s_));
  static const double bidiag_min = [] {  // RTLR_SVD_BIDIAG_MIN: smallest factor (entries) on the bidiagonal path
    const char* e = std::getenv("RTLR_SVD_BIDIAG_MIN");
    return e ? std::atof(e) : 0.0;
  }();
  if (!vectors && static_cast<double>(mrows) * ncols >= bidiag_min) {
    // singular values only (every outer iteration): bidiagonalisation of W
    // and Golub-Kahan multisection, without the QR and the Jacobi sweeps
    // (bidiag_coop2 + gk_multisect, tools/svd_time.py: 2048 x 600 56 -> 18.5
    // ms, 1152 x 403 28.5 -> 9.3, 512 x 178 8.6 -> 4.0, 128 x 64 3.0 -> 1.7;
    // RTLR_SVD_BIDIAG_MIN raises the size below which QR + Jacobi run)
    double* dsv = nrm_.ensure(std::max(ncols, 128));
    double* bw = work(bidiag_work_doubles(mrows, ncols));  // before work_.size(): argument order is unspecified
    if (bidiag_singular_values(mrows, ncols, Wm, mrows, dsv, bw, work_.size(), s_)) {
      ++svd_calls_;
      const double mm = static_cast<double>(mrows), nn = ncols;
      // 4 m n^2 - 4/3 n^3 flops; the factor crosses HBM once each way (its
      // per-column passes stay in L2)
      pt_.work(8.0 * 2.0 * mm * nn, 4.0 * mm * nn * nn - 4.0 / 3.0 * nn * nn * nn);
      std::vector<double> sv(ncols);
      RTLR_CUDA(cudaMemcpyAsync(sv.data(), dsv, ncols * sizeof(double), cudaMemcpyDeviceToHost, s_));
      RTLR_CUDA(cudaStreamSynchronize(s_));
      return sv;
    }
  }
  double* Q = svq_.ensure(static_cast<size_t>(mrows) * ncols);
  double* R = svr_.ensure(static_cast<size_t>(ncols) * ncols);
  double* Mt = svm_.ensure(static_cast<size_t>(ncols) * ncols);
  double* tau = tau_.ensure(ncols);
  // Singular values only (every outer iteration): R from the cooperative
  // QR; with vectors (the last iteration) the blocked QR forms Q too.
  if (vectors || !householder_r_coop(mrows, ncols, Wm, mrows, R, s_)) {
    double* qw = work(householder_qr_work(mrows, ncols));
    householder_qr(mrows, ncols, Wm, mrows, tau, Q, mrows, R, qw, work_.size(), s_);
  }
  transpose_kernel<<<g1(static_cast<long long>(ncols) * ncols), 256, 0, s_>>>(ncols, ncols, R, ncols, Mt, ncols);
  double* J = nullptr;
  if (vectors) {
    std::vector<double> eye(static_cast<size_t>(ncols) * ncols, 0.0);
    for (int i = 0; i < ncols; ++i) eye[i + static_cast<size_t>(i) * ncols] = 1.0;
    J = qq_.ensure(eye.size());
    RTLR_CUDA(cudaMemcpyAsync(J, eye.data(), eye.size() * sizeof(double), cudaMemcpyHostToDevice, s_));
  }
  int rotated = 0;
  int sweeps = 0;
  jacobi_svd(ncols, ncols, Mt, ncols, J, 60, &rotated, work(4096), s_, &sweeps);
  svd_sweeps_ += sweeps;
  {  // Householder R of the N_Omega x r (or r x N_Omega) factor, then one-sided
     // Jacobi sweeps on the n x n core (pair dots + rotations, 6 n^3 flops per sweep)
    const double mm = static_cast<double>(mrows), nn = ncols;
    pt_.work(8.0 * (2.0 * mm * nn + 2.0 * sweeps * nn * nn), 2.0 * mm * nn * nn - 2.0 / 3.0 * nn * nn * nn +
                                                                  6.0 * sweeps * nn * nn * nn);
  }
  ++svd_calls_;
  double* nr = nrm_.ensure(ncols);
  col_norms_kernel<<<ncols, 256, 0, s_>>>(ncols, ncols, Mt, ncols, nr);
  std::vector<double> sv(ncols);
  RTLR_CUDA(cudaMemcpyAsync(sv.data(), nr, ncols * sizeof(double), cudaMemcpyDeviceToHost, s_));
  RTLR_CUDA(cudaStreamSynchronize(s_));
  std::vector<int> order(ncols);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return sv[a] > sv[b]; });
  std::vector<double> s(ncols);
  for (int k = 0; k < ncols; ++k) s[k] = sv[order[k]];
  if (vectors && keep > 0) {
    // left singular vectors of W: Q J (mrows); right: the rotated columns of R^T / s (ncols)
    double* QJ = ybuf_.ensure(static_cast<size_t>(mrows) * ncols);
    gemm_nn(mrows, ncols, ncols, Q, mrows, J, ncols, QJ, mrows, s_);
    std::vector<double> hQJ(static_cast<size_t>(mrows) * ncols), hM(static_cast<size_t>(ncols) * ncols);
    RTLR_CUDA(cudaMemcpyAsync(hQJ.data(), QJ, hQJ.size() * sizeof(double), cudaMemcpyDeviceToHost, s_));
    RTLR_CUDA(cudaMemcpyAsync(hM.data(), Mt, hM.size() * sizeof(double), cudaMemcpyDeviceToHost, s_));
    RTLR_CUDA(cudaStreamSynchronize(s_));
    // U_C (r x keep) and V_C (N_Omega x keep), sorted: C = W^T = L S (Q J)^T (on_ct), else C = W
    std::vector<double> U(static_cast<size_t>(r) * keep, 0.0), V(static_cast<size_t>(nomega_) * keep, 0.0);
    for (int kk = 0; kk < keep; ++kk) {
      const int k = order[kk];
      const double sk = sv[k];
      for (int i = 0; i < ncols; ++i) {
        const double l = sk > 0.0 ? hM[i + static_cast<size_t>(k) * ncols] / sk : (i == kk ? 1.0 : 0.0);
        if (on_ct)
          U[i + static_cast<size_t>(kk) * r] = l;
        else
          V[i + static_cast<size_t>(kk) * nomega_] = l;
      }
      for (long long i = 0; i < mrows; ++i) {
        const double q = hQJ[i + static_cast<size_t>(k) * mrows];
        if (on_ct)
          V[i + static_cast<size_t>(kk) * nomega_] = q;
        else
          U[i + static_cast<size_t>(kk) * r] = q;
      }
    }
    // X_out = X U[:, :keep] on the device
    double* dU = gbuf_.ensure(U.size());
    RTLR_CUDA(cudaMemcpyAsync(dU, U.data(), U.size() * sizeof(double), cudaMemcpyHostToDevice, s_));
    double* dX = ybuf_.ensure(static_cast<size_t>(n_) * keep);
    gemm_nn(n_, keep, r, X_.col(0), X_.ld, dU, r, dX, n_, s_);
    Xout->resize(static_cast<size_t>(n_) * keep);
    RTLR_CUDA(cudaMemcpyAsync(Xout->data(), dX, Xout->size() * sizeof(double), cudaMemcpyDeviceToHost, s_));
    RTLR_CUDA(cudaStreamSynchronize(s_));
    *Vout = std::move(V);
  }
  return s;
}

// report.cpp:47-58: the reconstruction X diag(S) V^T is formed 128 angles at
// a time (as the reference's block loop), never whole.
double Problem::psi_difference(const double* d_psi, const double* d_X, const double* d_S, const double* d_V,
                               int r) {
  const long long n = hp_.ndof;
  const int nom = hp_.n_omega, block = 128, parts = 296;
  if (r < 0) throw std::invalid_argument("psi_difference: negative rank");
  // SV^T = diag(S) V^T (r x N_Omega), on the host from the device factors
  std::vector<double> S(r), V(static_cast<size_t>(nom) * r), svt(static_cast<size_t>(r) * nom);
  if (r > 0) {
    RTLR_CUDA(cudaMemcpyAsync(S.data(), d_S, r * sizeof(double), cudaMemcpyDeviceToHost, stream_));
    RTLR_CUDA(cudaMemcpyAsync(V.data(), d_V, V.size() * sizeof(double), cudaMemcpyDeviceToHost, stream_));
    RTLR_CUDA(cudaStreamSynchronize(stream_));
  }
  for (int j = 0; j < nom; ++j)
    for (int k = 0; k < r; ++k) svt[k + static_cast<size_t>(j) * r] = S[k] * V[j + static_cast<size_t>(k) * nom];
  DBuf<double> dsvt, rec, part;
  dsvt.upload(svt.data(), svt.size(), stream_);
  double* Y = rec.ensure(static_cast<size_t>(n) * block);
  double* pp = part.ensure(parts);
  std::vector<double> hp(parts);
  double acc = 0.0;
  for (int j0 = 0; j0 < nom; j0 += block) {
    const int nb = std::min(block, nom - j0);
    gemm_nn(n, nb, r, d_X, n, dsvt.get() + static_cast<size_t>(j0) * r, r, Y, n, stream_);
    sqdiff_partials<<<parts, 256, 0, stream_>>>(n, nb, d_psi + static_cast<size_t>(j0) * n, n, Y, n, pp);
    RTLR_CUDA(cudaGetLastError());
    RTLR_CUDA(cudaMemcpyAsync(hp.data(), pp, parts * sizeof(double), cudaMemcpyDeviceToHost, stream_));
    RTLR_CUDA(cudaStreamSynchronize(stream_));
    for (double v : hp) acc += v;  // fixed order
  }
  return std::sqrt(acc);
}

// proj/src/low_rank.cpp:436-492
SolveReport Problem::solve_low_rank(const LowRankOptions& o) {
  require_k1("solve_low_rank");
  if (o.use_dsa && sip_.get() == nullptr)
    throw std::invalid_argument("solve_low_rank: DSA requested but no diffusion system");
  const size_t n = hp_.ndof;
  SolveReport rep;
  rep.method = "lowrank";
  SubsampleRng rng(o.seed);
  RTLR_CUDA(cudaStreamSynchronize(stream_));
  const auto t0 = std::chrono::steady_clock::now();
  LowRankEngine eng(*this, o.inner);
  double* base = scratch_.ensure(3 * n);
  double *phi = base, *delta = base + n;
  RTLR_CUDA(cudaMemsetAsync(phi, 0, n * sizeof(double), stream_));
  InnerResult inner;
  int final_rank = 0;
  for (int it = 1; it <= o.max_iterations; ++it) {
    inner = eng.inner(phi, rng);
    eng.pt_.start("svd");
    const std::vector<double> sv = eng.svd(false, 0, nullptr, nullptr);
    eng.pt_.stop();
    const int rp = truncation_rank(sv, o.inner.eps_svd);
    diff_norms(static_cast<int>(n), eng.phi(), phi, norm_work_.get(), norm_work_.get() + 2 * kNormParts, stream_);
    RTLR_CUDA(cudaMemcpyAsync(h_pin_, norm_work_.get() + 2 * kNormParts, 2 * sizeof(double), cudaMemcpyDeviceToHost,
                              stream_));
    RTLR_CUDA(cudaStreamSynchronize(stream_));
    OuterRecord rec;
    rec.diff_two_norm = h_pin_[0];
    rec.diff_inf_norm = h_pin_[1];
    rec.rank = rp;
    rec.oversampling = rp > 0 ? static_cast<double>(inner.rank - rp) / rp : 0.0;
    rec.inner_iterations = inner.iterations;
    rec.sampled_count = inner.sampled_count;
    rec.fullrank_fallback = inner.exhausted;
    rep.sampled_log.push_back(inner.sampled_order);
    rep.iterations = it;
    final_rank = rp;
    if (rec.diff_inf_norm <= o.eps_si_sa) {
      rep.history.push_back(rec);
      rep.converged = true;
      RTLR_CUDA(cudaMemcpyAsync(phi, eng.phi(), n * sizeof(double), cudaMemcpyDeviceToDevice, stream_));
      break;
    }
    if (o.use_dsa) {
      eng.pt_.start("dsa");
      rec.dsa_iterations = dsa_correct(eng.phi(), phi, delta);
      // per PCG iteration: the SIP SpMV (5 4x4 blocks per cell), the V-cycle
      // (two block smoothing sweeps, transfers, coarser 5-point levels) and
      // the vector updates: ~2.5 KB and ~1.3 kflop per cell
      eng.pt_.work(2500.0 * hp_.ncell * rec.dsa_iterations, 1300.0 * hp_.ncell * rec.dsa_iterations);
      vadd(static_cast<int>(n), eng.phi(), delta, phi, stream_);
      eng.pt_.stop();
    } else {
      RTLR_CUDA(cudaMemcpyAsync(phi, eng.phi(), n * sizeof(double), cudaMemcpyDeviceToDevice, stream_));
    }
    rep.history.push_back(rec);
  }
  if (!rep.converged)
    RTLR_CUDA(cudaMemcpyAsync(phi, eng.phi(), n * sizeof(double), cudaMemcpyDeviceToDevice, stream_));
  if (eng.pf_check_worst_ > 0.0)
    std::fprintf(stderr, "[rtlr prefactor] bordered vs full pivoted LU over %lld candidate batches: worst relative difference of a solution %.3e\n",
                 eng.pf_used_, eng.pf_check_worst_);
  if (eng.pt_.on) {
    std::fprintf(stderr, "[rtlr profile] low-rank phases (s):");
    for (auto& e : eng.pt_.acc) std::fprintf(stderr, " %s=%.4f", e.first.c_str(), e.second);
    std::fprintf(stderr,
                 " | reorth: %d rebuilds, %.4f s (inside cgs) | cgs: block %.4f (GEMMs %.4f), per-snapshot %.4f | svd: %d calls, "
                 "%d Jacobi sweeps | galerkin: %lld batches, %lld systems (prefactored %lld, fell back %lld) | verify: %lld passes, %lld angles | "
                 "device allocations (process): %lld (%lld reused), %.1f GB, %.4f s (free %.4f, malloc %.4f)\n",
                 eng.reorth_count_, eng.reorth_seconds_, eng.cgs_split_[0], eng.cgs_split_[3], eng.cgs_split_[1], eng.svd_calls_,
                 eng.svd_sweeps_, eng.gal_calls_, eng.gal_systems_, eng.pf_used_, eng.pf_missed_, eng.verify_calls_, eng.verify_angles_,
                 alloc_stats().count, alloc_stats().reused, alloc_stats().bytes / 1e9, alloc_stats().seconds,
                 alloc_stats().free_s,
                 alloc_stats().malloc_s);
  }
  rep.phase_work.assign(4 * kPhaseCount, 0.0);
  for (int k = 0; k < kPhaseCount; ++k) {
    rep.phase_work[4 * k] = eng.pt_.seconds(k);
    rep.phase_work[4 * k + 1] = eng.pt_.bytes[k];
    rep.phase_work[4 * k + 2] = eng.pt_.flops[k];
    rep.phase_work[4 * k + 3] = static_cast<double>(eng.pt_.calls[k]);
  }
  rep.phi.resize(n);
  RTLR_CUDA(cudaMemcpyAsync(rep.phi.data(), phi, n * sizeof(double), cudaMemcpyDeviceToHost, stream_));
  RTLR_CUDA(cudaStreamSynchronize(stream_));
  rep.psi_dofs = static_cast<long long>(final_rank) * (static_cast<long long>(n) + hp_.n_omega);
  if (o.build_factors) {
    // truncate_factors (low_rank.cpp:268-277) on the last inner loop's C, X
    const std::vector<double> sv = eng.svd(false, 0, nullptr, nullptr);
    const int r = truncation_rank(sv, o.inner.eps_svd);
    std::vector<double> Xo, Vo;
    const std::vector<double> s2 = eng.svd(true, r, &Xo, &Vo);
    rep.has_factors = true;
    rep.factors.rank = r;
    rep.factors.S.assign(s2.begin(), s2.begin() + r);
    rep.factors.X = std::move(Xo);
    rep.factors.V = std::move(Vo);
  }
  rep.solve_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return rep;
}

}  // namespace cuda
}  // namespace rtlr
