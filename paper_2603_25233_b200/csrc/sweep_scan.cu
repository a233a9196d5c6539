// K1 — batched transport sweep, row-scan formulation (replaces rtlr::sweep,
// proj/src/sweep.cpp:9-57).
//
// The upwind DG couplings of K = 1 are rank one per axis (b^- = -t_L t_R^T,
// operators.cpp:47-57): a cell sees its x-upwind neighbour only through the
// two outflow-trace coefficients tau (one per y-mode).  Along a mesh row the
// x dependence is therefore a 2-dimensional affine recurrence
//     tau_a = G_a tau_{a-1} + f_a,
//     f_a = T_x M_a^-1 (rhs_a - Omega_y B_y psi_{a,b-1}),  G_a = -T_x M_a^-1 K_x,
// and psi_a = M_a^-1 (rhs_a - K_x tau_{a-1} - ...).  A warp processes a row
// in chunks of 64 consecutive cells, two adjacent cells per lane (so every
// warp-wide load/store covers one contiguous 2 KB segment), composes its two
// cells' maps locally and resolves the recurrence across the lanes with a
// 5-level branch-free shuffle scan of affine maps; the carry tau passes from
// chunk to chunk.  Rows run in upwind order; the y-upwind traces of the
// previous row live in a per-warp trace line (two planes, one per x-mode;
// shared memory, or L2 for very wide rows).  Sources stream in one chunk
// ahead through registers and kAhead chunks ahead through bulk L2 prefetches.
// With W > 1 warps per direction, warp w owns rows w, w+W, ... and reads the
// line of warp w-1 behind a per-chunk progress counter (data-ready waits
// only, along the sweep DAG: no cycles).
//
// Uniform media (every Sigma_t block bitwise equal) use one per-direction
// inverse M^-1, so G is constant and only the 2-vector f is scanned; general
// media factor each cell block with the reference's partial-pivot LU
// (first maximum, singular test min|U_ii| <= 1e-14 max|block|) and scan the
// full affine maps.
#include <algorithm>
#include <cmath>

#include "device.cuh"

namespace rtlr {
namespace cuda {

namespace {

#define A_(i, j) A[(j) * 4 + (i)]

template <int K>
__device__ __forceinline__ void pivot_rows_n(double* A, double* b0, double* b1, double* b2, int p) {
#pragma unroll
  for (int i = K + 1; i < 4; ++i) {
    const bool s = (p == i);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const double x = A_(K, j), y = A_(i, j);
      A_(K, j) = s ? y : x;
      A_(i, j) = s ? x : y;
    }
    double x = b0[K], y = b0[i];
    b0[K] = s ? y : x;
    b0[i] = s ? x : y;
    x = b1[K], y = b1[i];
    b1[K] = s ? y : x;
    b1[i] = s ? x : y;
    x = b2[K], y = b2[i];
    b2[K] = s ? y : x;
    b2[i] = s ? x : y;
  }
}

template <int K>
__device__ __forceinline__ int argmax_col_n(const double* A) {
  int p = K;
  double big = fabs(A_(K, K));
#pragma unroll
  for (int i = K + 1; i < 4; ++i) {
    const double v = fabs(A_(i, K));
    if (v > big) {
      big = v;
      p = i;
    }
  }
  return p;
}

template <int K>
__device__ __forceinline__ void eliminate_n(double* A, double* b0, double* b1, double* b2) {
  const double inv = 1.0 / A_(K, K);
#pragma unroll
  for (int i = K + 1; i < 4; ++i) {
    const double l = A_(i, K) * inv;
#pragma unroll
    for (int j = K + 1; j < 4; ++j) A_(i, j) -= l * A_(K, j);
    b0[i] -= l * b0[K];
    b1[i] -= l * b1[K];
    b2[i] -= l * b2[K];
  }
}

__device__ __forceinline__ void backsub(const double* A, double* b) {
#pragma unroll
  for (int i = 3; i >= 0; --i) {
    b[i] = b[i] / A_(i, i);
#pragma unroll
    for (int j = 0; j < i; ++j) b[j] -= b[i] * A_(j, i);
  }
}

// Solves A [x0 x1 x2] = [b0 b1 b2] with one partial-pivot LU (first
// maximum); false on the reference's singular test (sweep.cpp:49-52).
__device__ __forceinline__ bool lu_solve4x3(double* A, double* b0, double* b1, double* b2) {
  double amax = 0.0;
#pragma unroll
  for (int k = 0; k < 16; ++k) amax = fmax(amax, fabs(A[k]));
  int p = argmax_col_n<0>(A);
  pivot_rows_n<0>(A, b0, b1, b2, p);
  eliminate_n<0>(A, b0, b1, b2);
  p = argmax_col_n<1>(A);
  pivot_rows_n<1>(A, b0, b1, b2, p);
  eliminate_n<1>(A, b0, b1, b2);
  p = argmax_col_n<2>(A);
  pivot_rows_n<2>(A, b0, b1, b2, p);
  eliminate_n<2>(A, b0, b1, b2);
  const double dmin = fmin(fmin(fabs(A_(0, 0)), fabs(A_(1, 1))), fmin(fabs(A_(2, 2)), fabs(A_(3, 3))));
  backsub(A, b0);
  backsub(A, b1);
  backsub(A, b2);
  return dmin > 1e-14 * amax;
}

#undef A_

__device__ __forceinline__ void ld_cell256(const double* p, double v[4]) {
  asm volatile("ld.global.nc.L2::256B.v4.f64 {%0, %1, %2, %3}, [%4];"
               : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
               : "l"(p));
}
__device__ __forceinline__ void st_cell256(double* p, const double v[4]) {
  asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(v[0]), "d"(v[1]), "d"(v[2]),
               "d"(v[3])
               : "memory");
}
// Bulk prefetch of [p, p + bytes) into L2 (one instruction per chunk).
__device__ __forceinline__ void prefetch_l2(const double* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
// Trace-line access: explicit shared-memory or L2 (.cg) instructions, so the
// compiler never falls back to generic loads for the smem case.
__device__ __forceinline__ double2 ld_line(const double* p, bool smem) {
  double2 v;
  if (smem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(p));
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(s) : "memory");
  } else {
    asm volatile("ld.global.cg.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p) : "memory");
  }
  return v;
}
__device__ __forceinline__ void st_line(double* p, double x, double y, bool smem) {
  if (smem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(p));
    asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(s), "d"(x), "d"(y) : "memory");
  } else {
    asm volatile("st.global.cg.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(x), "d"(y) : "memory");
  }
}

constexpr int kLineSmemBudget = 96 * 1024;  // bytes of trace lines per block kept in smem
constexpr int kWarps = 8;                   // warps per block
constexpr int kCpl = 2;                     // adjacent cells per lane
constexpr int kChunk = 32 * kCpl;           // cells per warp step
constexpr int kAhead = 4;                   // chunks prefetched into L2 ahead of the sweep

// Per-direction constants (shared memory, written by warp 0 of the group):
//   [0..16)   M^-1 (uniform) or Omega_x Ax + Omega_y Ay (general), column-major
//   [16..24)  kx[2] tx[2] ky[2] ty[2]
//   [24..32)  Q = -M^-1 K_x (4 x 2, uniform)
//   [32..36)  G = T_x Q (2 x 2, uniform)
//   [36..164) G^(2(l+1)), l = 0..31 (uniform): the map of 2(l+1) cells
constexpr int kKT = 16, kQ = 24, kG = 32, kGP = 36, kConsts = 164;

// Doubles per trace plane (even, so both planes stay 16-byte aligned).
__host__ __device__ constexpr int line_pitch(int nx) { return (nx + 1) & ~1; }
__host__ __device__ constexpr int group_doubles(int W, int nx, bool smem_lines) {
  return kConsts + 2 * ((W + 3) / 4) + (smem_lines ? W * 2 * line_pitch(nx) : 0);
}

struct Group {
  double* c;           // kConsts
  volatile int* prod;  // W progress counters (chunks published)
  double* lines;       // W x 2 planes x pitch
};

__device__ __forceinline__ void mat2_vec(const double* G, double x0, double x1, double& y0, double& y1) {
  y0 = G[0] * x0 + G[2] * x1;  // column-major 2 x 2
  y1 = G[1] * x0 + G[3] * x1;
}

template <bool UNIFORM, bool MULTI, bool HAS_BC>
__global__ void __launch_bounds__(256, 2) sweep_scan_kernel(const SweepArgs a, int W, bool smem_lines) {
  extern __shared__ double smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int groups = kWarps / W;
  const int g = wib / W, w = wib % W;
  const int slot = blockIdx.x * groups + g;
  if (slot >= a.n) return;  // a whole direction group exits together
  const int nx = a.nx, ny = a.ny;
  const int pitch = line_pitch(nx);
  Group G;
  {
    double* base = smem + static_cast<size_t>(g) * group_doubles(W, nx, smem_lines);
    G.c = base;
    G.prod = reinterpret_cast<int*>(base + kConsts);
    G.lines = smem_lines ? base + kConsts + 2 * ((W + 3) / 4)
                         : a.line + static_cast<size_t>(slot) * W * 2 * pitch;
  }
  const int ang = a.angles ? a.angles[slot] : slot;
  const double omx = a.dirs[3 * ang], omy = a.dirs[3 * ang + 1];
  const bool xu = omx >= 0.0, yu = omy >= 0.0;  // sweep.cpp:37-38
  if (w == 0) {
    const double* ax = xu ? a.sc.ax_minus : a.sc.ax_plus;
    const double* ay = yu ? a.sc.ay_minus : a.sc.ay_plus;
    if (lane < 16) {
      const double d = omx * ax[lane] + omy * ay[lane];
      G.c[lane] = UNIFORM ? d + a.sigma_t[lane] : d;
    }
    if (lane < 2) {
      // (B psi_up)[my,mx] = c[mx] (t . psi_up[my,:]), (c,t) = (-t_L,t_R) minus / (t_R,t_L) plus
      G.c[kKT + lane] = omx * (xu ? -a.sc.trx_l[lane] : a.sc.trx_r[lane]);
      G.c[kKT + 2 + lane] = xu ? a.sc.trx_r[lane] : a.sc.trx_l[lane];
      G.c[kKT + 4 + lane] = omy * (yu ? -a.sc.try_l[lane] : a.sc.try_r[lane]);
      G.c[kKT + 6 + lane] = yu ? a.sc.try_r[lane] : a.sc.try_l[lane];
    }
    __syncwarp();
    if (UNIFORM && lane == 0) {
      // M^-1 columns via the reference LU; Q = -M^-1 K_x; G = T_x Q; (G^2)^(l+1)
      double Mi[16];
      for (int c = 0; c < 4; c += 3) {
        double A[16], e0[4] = {0, 0, 0, 0}, e1[4] = {0, 0, 0, 0}, e2[4] = {0, 0, 0, 0};
        for (int k = 0; k < 16; ++k) A[k] = G.c[k];
        e0[c] = 1.0;
        if (c + 1 < 4) e1[c + 1] = 1.0;
        if (c + 2 < 4) e2[c + 2] = 1.0;
        if (!lu_solve4x3(A, e0, e1, e2)) atomicExch(a.err, 1);
        for (int r = 0; r < 4; ++r) {
          Mi[c * 4 + r] = e0[r];
          if (c + 1 < 4) Mi[(c + 1) * 4 + r] = e1[r];
          if (c + 2 < 4) Mi[(c + 2) * 4 + r] = e2[r];
        }
      }
      const double kx0 = G.c[kKT], kx1 = G.c[kKT + 1], tx0 = G.c[kKT + 2], tx1 = G.c[kKT + 3];
      // K_x (4 x 2): column my has kx[mx] at rows (my, mx)
      double Q[8];
      for (int my = 0; my < 2; ++my)
        for (int r = 0; r < 4; ++r)
          Q[my * 4 + r] = -(Mi[(my * 2 + 0) * 4 + r] * kx0 + Mi[(my * 2 + 1) * 4 + r] * kx1);
      // G = T_x Q (2 x 2): row m = tx . Q[(m,0..1), :]
      double Gm[4];
      for (int col = 0; col < 2; ++col)
        for (int m = 0; m < 2; ++m) Gm[col * 2 + m] = tx0 * Q[col * 4 + m * 2] + tx1 * Q[col * 4 + m * 2 + 1];
      for (int k = 0; k < 16; ++k) G.c[k] = Mi[k];
      for (int k = 0; k < 8; ++k) G.c[kQ + k] = Q[k];
      for (int e = 0; e < 4; ++e) G.c[kG + e] = Gm[e];
      double G2[4];
      for (int col = 0; col < 2; ++col)
        for (int m = 0; m < 2; ++m) G2[col * 2 + m] = Gm[m] * Gm[col * 2] + Gm[2 + m] * Gm[col * 2 + 1];
      double P[4] = {G2[0], G2[1], G2[2], G2[3]};
      for (int k = 0; k < 32; ++k) {
        for (int e = 0; e < 4; ++e) G.c[kGP + 4 * k + e] = P[e];
        double N[4];
        for (int col = 0; col < 2; ++col)
          for (int m = 0; m < 2; ++m) N[col * 2 + m] = G2[m] * P[col * 2] + G2[2 + m] * P[col * 2 + 1];
        for (int e = 0; e < 4; ++e) P[e] = N[e];
      }
    }
    if (lane < W) G.prod[lane] = 0;
  }
  asm volatile("bar.sync %0, %1;" ::"r"(g + 1), "r"(W * 32) : "memory");

  const double* cst = G.c;
  const double kx0 = cst[kKT], kx1 = cst[kKT + 1], tx0 = cst[kKT + 2], tx1 = cst[kKT + 3];
  const double ky0 = cst[kKT + 4], ky1 = cst[kKT + 5], ty0 = cst[kKT + 6], ty1 = cst[kKT + 7];

  const int nchunk = (nx + kChunk - 1) / kChunk;
  const int nrows = (ny - w + W - 1) / W;  // rows w, w+W, ... of this warp
  const int nsteps = nrows * nchunk;
  const double* rhs = a.rhs + static_cast<long long>(slot) * a.rhs_stride;
  const double* bc = HAS_BC ? a.bc + static_cast<long long>(ang) * a.bc_stride : nullptr;
  double* psi = a.psi + static_cast<long long>(slot) * a.psi_stride;
  const int pw = (w + W - 1) % W;
  double* my_line = G.lines + static_cast<size_t>(w) * 2 * pitch;
  const double* in_line = G.lines + static_cast<size_t>(pw) * 2 * pitch;
  const int c0 = kCpl * lane;  // this lane's first sweep column within a chunk

  auto row_base = [&](int rowk) -> long long {
    const int r = w + rowk * W;
    return static_cast<long long>(yu ? r : ny - 1 - r) * nx;
  };
  // cell of sweep column col (clamped to a valid cell past the row end)
  auto cell_of = [&](long long row0, int col) -> long long {
    return row0 + (col < nx ? (xu ? col : nx - 1 - col) : 0);
  };
  auto prefetch_chunk = [&](int rowk, int k) {
    const long long r0 = row_base(rowk);
    const int lo = k * kChunk, cnt = min(kChunk, nx - lo);
    const long long first = xu ? r0 + lo : r0 + nx - lo - cnt;
    prefetch_l2(rhs + 4 * first, static_cast<unsigned>(cnt) * 32u);
    if (HAS_BC) prefetch_l2(bc + 4 * first, static_cast<unsigned>(cnt) * 32u);
  };

  int prow = 0, pk = 0;  // L2 prefetch position, kAhead chunks in front
  if (lane == 0) {
    for (int t = 0; t < kAhead + 1 && prow < nrows; ++t) {
      prefetch_chunk(prow, pk);
      if (++pk == nchunk) pk = 0, ++prow;
    }
  }
  double nv0[4], nv1[4];  // next step's sources
  long long row0 = row_base(0);
  ld_cell256(rhs + 4 * cell_of(row0, c0), nv0);
  ld_cell256(rhs + 4 * cell_of(row0, c0 + 1), nv1);

  int rowk = 0, k = 0;
  double tc0 = 0.0, tc1 = 0.0;  // x-trace carry into the chunk
  for (int t = 0; t < nsteps; ++t) {
    if (k == 0) tc0 = tc1 = 0.0;  // vacuum x-inflow at the row start
    const int col = k * kChunk + c0;
    const bool act0 = col < nx, act1 = col + 1 < nx;
    const long long cell0 = cell_of(row0, col), cell1 = cell_of(row0, col + 1);
    double v0[4], v1[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v0[i] = nv0[i];
      v1[i] = nv1[i];
    }
    int nk = k + 1, nrowk = rowk;
    long long nrow0 = row0;
    if (nk == nchunk) {
      nk = 0;
      ++nrowk;
      if (nrowk < nrows) nrow0 = row_base(nrowk);
    }
    if (t + 1 < nsteps) {
      const int ncol = nk * kChunk + c0;
      ld_cell256(rhs + 4 * cell_of(nrow0, ncol), nv0);
      ld_cell256(rhs + 4 * cell_of(nrow0, ncol + 1), nv1);
    }
    if (lane == 0 && prow < nrows) {
      prefetch_chunk(prow, pk);
      if (++pk == nchunk) pk = 0, ++prow;
    }
    if (HAS_BC) {
      double g0[4], g1[4];
      ld_cell256(bc + 4 * cell0, g0);
      ld_cell256(bc + 4 * cell1, g1);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        v0[i] += g0[i];
        v1[i] += g1[i];
      }
    }
    // y-upwind traces (per x-mode) of these columns from the previous row
    double y00 = 0.0, y01 = 0.0, y10 = 0.0, y11 = 0.0;  // y{cell}{x-mode}
    const int r = w + rowk * W;
    if (r > 0) {
      if (MULTI) {
        if (lane == 0) {
          const int need = (w == 0 ? rowk - 1 : rowk) * nchunk + k + 1;
          while (G.prod[pw] < need) {
          }
          __threadfence_block();
        }
        __syncwarp();
      }
      if (act0) {
        const double2 p0 = ld_line(in_line + col, smem_lines);
        const double2 p1 = ld_line(in_line + pitch + col, smem_lines);
        y00 = p0.x;
        y01 = p1.x;
        y10 = act1 ? p0.y : 0.0;  // the padding column of an odd row is never written
        y11 = act1 ? p1.y : 0.0;
      }
    }
    // local = rhs - Omega_y By psi_y   (the x term enters through the scan)
    v0[0] -= ky0 * y00;
    v0[1] -= ky0 * y01;
    v0[2] -= ky1 * y00;
    v0[3] -= ky1 * y01;
    v1[0] -= ky0 * y10;
    v1[1] -= ky0 * y11;
    v1[2] -= ky1 * y10;
    v1[3] -= ky1 * y11;

    double ps0[4], ps1[4];
    // Constants are re-read from shared memory every step as 16-byte
    // broadcasts (one wavefront each); registers hold only the stream state.
    const double2* c2 = reinterpret_cast<const double2*>(cst);
    if (UNIFORM) {
      double u0[4], u1[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {  // u = M^-1 v, column by column
        const double2 lo = c2[2 * c], hi = c2[2 * c + 1];
        if (c == 0) {
          u0[0] = lo.x * v0[0], u0[1] = lo.y * v0[0], u0[2] = hi.x * v0[0], u0[3] = hi.y * v0[0];
          u1[0] = lo.x * v1[0], u1[1] = lo.y * v1[0], u1[2] = hi.x * v1[0], u1[3] = hi.y * v1[0];
        } else {
          u0[0] += lo.x * v0[c], u0[1] += lo.y * v0[c], u0[2] += hi.x * v0[c], u0[3] += hi.y * v0[c];
          u1[0] += lo.x * v1[c], u1[1] += lo.y * v1[c], u1[2] += hi.x * v1[c], u1[3] += hi.y * v1[c];
        }
      }
      // f = T_x u (per y-mode); lane map over its two cells: tau -> G^2 tau + (G f0 + f1).
      // The chunk's carry enters lane 0's map before the scan, so the
      // inclusive scan yields tau after each lane's last cell directly.
      const double f00 = tx0 * u0[0] + tx1 * u0[1], f01 = tx0 * u0[2] + tx1 * u0[3];
      const double f10 = tx0 * u1[0] + tx1 * u1[1], f11 = tx0 * u1[2] + tx1 * u1[3];
      const double2 g01 = c2[kG / 2], g23 = c2[kG / 2 + 1];
      double s0 = f10 + g01.x * f00 + g23.x * f01;
      double s1 = f11 + g01.y * f00 + g23.y * f01;
      {
        const double2 p01 = c2[kGP / 2], p23 = c2[kGP / 2 + 1];  // G^2
        const double t0 = lane == 0 ? tc0 : 0.0, t1 = lane == 0 ? tc1 : 0.0;
        s0 += p01.x * t0 + p23.x * t1;
        s1 += p01.y * t0 + p23.y * t1;
      }
      // inclusive scan over the lanes: s_l <- s_l + G^(2d) s_{l-d}
#pragma unroll
      for (int l = 0; l < 5; ++l) {
        const int d = 1 << l;
        double o0 = __shfl_up_sync(0xffffffffu, s0, d);
        double o1 = __shfl_up_sync(0xffffffffu, s1, d);
        o0 = lane >= d ? o0 : 0.0;
        o1 = lane >= d ? o1 : 0.0;
        const double2 p01 = c2[(kGP + 4 * (d - 1)) / 2], p23 = c2[(kGP + 4 * (d - 1)) / 2 + 1];
        s0 += p01.x * o0 + p23.x * o1;
        s1 += p01.y * o0 + p23.y * o1;
      }
      double ti0 = __shfl_up_sync(0xffffffffu, s0, 1), ti1 = __shfl_up_sync(0xffffffffu, s1, 1);
      if (lane == 0) ti0 = tc0, ti1 = tc1;
      tc0 = __shfl_sync(0xffffffffu, s0, 31);
      tc1 = __shfl_sync(0xffffffffu, s1, 31);
      // psi = u + Q tau_in, cell by cell
      const double m0 = f00 + g01.x * ti0 + g23.x * ti1, m1 = f01 + g01.y * ti0 + g23.y * ti1;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const double2 qa = c2[kQ / 2 + h], qb = c2[kQ / 2 + 2 + h];  // Q[2h..2h+1], Q[4+2h..]
        ps0[2 * h] = u0[2 * h] + qa.x * ti0 + qb.x * ti1;
        ps0[2 * h + 1] = u0[2 * h + 1] + qa.y * ti0 + qb.y * ti1;
        ps1[2 * h] = u1[2 * h] + qa.x * m0 + qb.x * m1;
        ps1[2 * h + 1] = u1[2 * h + 1] + qa.y * m0 + qb.y * m1;
      }
    } else {
      // per cell: [u | Qc] = M_a^-1 [local | -K_x], G_a = T_x Qc, f_a = T_x u
      double Qc0[8], Qc1[8];
      bool ok0, ok1;
      {
        double A[16];
        const double2* sb = reinterpret_cast<const double2*>(a.sigma_t + 16 * cell0);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const double2 s2 = __ldg(sb + e), m2 = c2[e];
          A[2 * e] = m2.x + s2.x;
          A[2 * e + 1] = m2.y + s2.y;
        }
        double b1[4] = {-kx0, -kx1, 0.0, 0.0}, b2[4] = {0.0, 0.0, -kx0, -kx1};
        ok0 = lu_solve4x3(A, v0, b1, b2);
#pragma unroll
        for (int i = 0; i < 4; ++i) Qc0[i] = b1[i], Qc0[4 + i] = b2[i];
      }
      {
        double A[16];
        const double2* sb = reinterpret_cast<const double2*>(a.sigma_t + 16 * cell1);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const double2 s2 = __ldg(sb + e), m2 = c2[e];
          A[2 * e] = m2.x + s2.x;
          A[2 * e + 1] = m2.y + s2.y;
        }
        double b1[4] = {-kx0, -kx1, 0.0, 0.0}, b2[4] = {0.0, 0.0, -kx0, -kx1};
        ok1 = lu_solve4x3(A, v1, b1, b2);
#pragma unroll
        for (int i = 0; i < 4; ++i) Qc1[i] = b1[i], Qc1[4 + i] = b2[i];
      }
      if ((!ok0 && act0) || (!ok1 && act1)) atomicExch(a.err, 1);
      double G0[4], G1[4];
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        G0[c * 2 + 0] = tx0 * Qc0[c * 4 + 0] + tx1 * Qc0[c * 4 + 1];
        G0[c * 2 + 1] = tx0 * Qc0[c * 4 + 2] + tx1 * Qc0[c * 4 + 3];
        G1[c * 2 + 0] = tx0 * Qc1[c * 4 + 0] + tx1 * Qc1[c * 4 + 1];
        G1[c * 2 + 1] = tx0 * Qc1[c * 4 + 2] + tx1 * Qc1[c * 4 + 3];
      }
      const double f00 = tx0 * v0[0] + tx1 * v0[1], f01 = tx0 * v0[2] + tx1 * v0[3];
      const double f10 = tx0 * v1[0] + tx1 * v1[1], f11 = tx0 * v1[2] + tx1 * v1[3];
      // lane map (A, s) = (G1 G0, G1 f0 + f1)
      double A0, A1, A2, A3, s0, s1;
      mat2_vec(G1, G0[0], G0[1], A0, A1);
      mat2_vec(G1, G0[2], G0[3], A2, A3);
      mat2_vec(G1, f00, f01, s0, s1);
      s0 += f10;
      s1 += f11;
      {  // the chunk's carry enters lane 0's map
        const double t0 = lane == 0 ? tc0 : 0.0, t1 = lane == 0 ? tc1 : 0.0;
        s0 += A0 * t0 + A2 * t1;
        s1 += A1 * t0 + A3 * t1;
      }
#pragma unroll
      for (int l = 0; l < 5; ++l) {
        const int d = 1 << l;
        const bool in = lane >= d;
        double p0 = __shfl_up_sync(0xffffffffu, A0, d), p1 = __shfl_up_sync(0xffffffffu, A1, d);
        double p2 = __shfl_up_sync(0xffffffffu, A2, d), p3 = __shfl_up_sync(0xffffffffu, A3, d);
        double o0 = __shfl_up_sync(0xffffffffu, s0, d), o1 = __shfl_up_sync(0xffffffffu, s1, d);
        p0 = in ? p0 : 1.0;
        p1 = in ? p1 : 0.0;
        p2 = in ? p2 : 0.0;
        p3 = in ? p3 : 1.0;
        o0 = in ? o0 : 0.0;
        o1 = in ? o1 : 0.0;
        // (A, s) <- (A, s) o (P, o) = (A P, A o + s)
        s0 += A0 * o0 + A2 * o1;
        s1 += A1 * o0 + A3 * o1;
        const double n0 = A0 * p0 + A2 * p1, n1 = A1 * p0 + A3 * p1;
        const double n2 = A0 * p2 + A2 * p3, n3 = A1 * p2 + A3 * p3;
        A0 = n0;
        A1 = n1;
        A2 = n2;
        A3 = n3;
      }
      double ti0 = __shfl_up_sync(0xffffffffu, s0, 1), ti1 = __shfl_up_sync(0xffffffffu, s1, 1);
      if (lane == 0) ti0 = tc0, ti1 = tc1;
      tc0 = __shfl_sync(0xffffffffu, s0, 31);
      tc1 = __shfl_sync(0xffffffffu, s1, 31);
#pragma unroll
      for (int i = 0; i < 4; ++i) ps0[i] = v0[i] + Qc0[i] * ti0 + Qc0[4 + i] * ti1;
      double m0, m1;
      mat2_vec(G0, ti0, ti1, m0, m1);
      m0 += f00;
      m1 += f01;
#pragma unroll
      for (int i = 0; i < 4; ++i) ps1[i] = v1[i] + Qc1[i] * m0 + Qc1[4 + i] * m1;
    }
    if (act0) {
      st_cell256(psi + 4 * cell0, ps0);
      if (act1) st_cell256(psi + 4 * cell1, ps1);
      // y-outflow traces (per x-mode) for the next row
      st_line(my_line + col, ty0 * ps0[0] + ty1 * ps0[2], ty0 * ps1[0] + ty1 * ps1[2], smem_lines);
      st_line(my_line + pitch + col, ty0 * ps0[1] + ty1 * ps0[3], ty0 * ps1[1] + ty1 * ps1[3], smem_lines);
    }
    if (MULTI) {
      __syncwarp();
      if (lane == 0) {
        __threadfence_block();
        G.prod[w] = t + 1;
      }
    } else {
      __syncwarp();  // own line: the next row reads what this row wrote
    }
    k = nk;
    rowk = nrowk;
    row0 = nrow0;
  }
}

int sm_count() {
  static const int n = [] {
    int d = 0, v = 148;
    if (cudaGetDevice(&d) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d);
    return v;
  }();
  return n;
}

}  // namespace

void launch_sweep_scan(const SweepArgs& a, bool uniform, cudaStream_t s) {
  if (a.n <= 0) return;
  const bool smem_lines =
      static_cast<size_t>(kWarps) * 2 * line_pitch(a.nx) * sizeof(double) <= kLineSmemBudget;
  // Warps per direction: the W in {1, 2, 4, 8} (at most one per 2 rows) whose
  // last wave of warps is fullest — the resident warp slots are
  // SMs x blocks/SM x kWarps; ties keep the smaller W.
  int W = 1;
  double best = -1.0;
  for (int c = 1; c <= kWarps && (c == 1 || 2 * c <= a.ny); c *= 2) {
    const size_t smem = static_cast<size_t>(kWarps / c) * group_doubles(c, a.nx, smem_lines) * sizeof(double);
    const int per_sm = std::max(1, std::min(2, static_cast<int>((227u * 1024u) / (smem + 1024u))));
    const double slots = static_cast<double>(sm_count()) * per_sm * kWarps;
    const double waves = static_cast<double>(a.n) * c / slots;
    const double eff = waves <= 1.0 ? waves : waves / std::ceil(waves);
    if (eff > best + 1e-3) {
      best = eff;
      W = c;
    }
  }
  const int groups = kWarps / W;
  const int blocks = (a.n + groups - 1) / groups;
  const size_t smem = static_cast<size_t>(groups) * group_doubles(W, a.nx, smem_lines) * sizeof(double);
  auto go = [&](auto kern) {
    RTLR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    kern<<<blocks, kWarps * 32, smem, s>>>(a, W, smem_lines);
  };
  const bool bc = a.bc != nullptr;
  if (uniform) {
    if (W > 1)
      bc ? go(sweep_scan_kernel<true, true, true>) : go(sweep_scan_kernel<true, true, false>);
    else
      bc ? go(sweep_scan_kernel<true, false, true>) : go(sweep_scan_kernel<true, false, false>);
  } else {
    if (W > 1)
      bc ? go(sweep_scan_kernel<false, true, true>) : go(sweep_scan_kernel<false, true, false>);
    else
      bc ? go(sweep_scan_kernel<false, false, true>) : go(sweep_scan_kernel<false, false, false>);
  }
  RTLR_CUDA(cudaGetLastError());
}

}  // namespace cuda
}  // namespace rtlr
