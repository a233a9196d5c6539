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
// 5-level shuffle scan of affine maps (predicated FMAs, no selects); the
// chunk's carry tau enters lane 0's map, so the scan yields every lane's tau
// directly.  Rows run in upwind order; the y-upwind traces of the previous
// row live in a per-warp trace line (two planes, one per x-mode; shared
// memory, or L2 for very wide rows).  Sources stream in one step ahead
// through registers (two register sets, the loop unrolled by two) and a few
// chunks ahead through bulk L2 prefetches.  With W > 1 warps per direction,
// warp w owns rows w, w+W, ... and reads the line of warp w-1 behind a
// per-chunk progress counter (acquire/release; data-ready waits only, along
// the sweep DAG: no cycles).
//
// The sweep loop is specialised on the x-direction sign, so cell addresses
// advance by a compile-time stride and a lane's second cell is an immediate
// +-32 B offset.  Everything per step is sized to keep SM-side work (issue
// slots, shared-memory wavefronts) low: the kernel must stay HBM-bound when
// the board power cap pulls the SM clock down under sustained load.
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
// Bulk prefetch of [p, p + bytes) into L2 (one instruction per unit).
__device__ __forceinline__ void prefetch_l2(const double* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
// Trace-line access: explicit shared-memory or L2 (.cg) instructions, so the
// compiler never falls back to generic loads for the smem case.
__device__ __forceinline__ double2 ld_line(const double* p, bool smem) {
  double2 v;
  if (smem) {
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(smem_u32(p)) : "memory");
  } else {
    asm volatile("ld.global.cg.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p) : "memory");
  }
  return v;
}
__device__ __forceinline__ void st_line(double* p, double x, double y, bool smem) {
  if (smem) {
    asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(smem_u32(p)), "d"(x), "d"(y) : "memory");
  } else {
    asm volatile("st.global.cg.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(x), "d"(y) : "memory");
  }
}
// Progress counters (shared memory), CTA-scope acquire/release: the
// producer and consumer warps share the CTA, whichever state space (shared
// memory or L2) holds the trace lines.
__device__ __forceinline__ void wait_progress(const int* p, int need) {
  int v;
  do {
    asm volatile("ld.acquire.cta.shared.b32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  } while (v < need);
}
__device__ __forceinline__ void publish_progress(int* p, int v) {
  asm volatile("st.release.cta.shared.b32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
// fp64 shuffles as two 32-bit shuffles on the register pair (keeps the
// compiler from reshuffling the halves).
__device__ __forceinline__ double shfl_up_f64(double x, int d) {
  double r;
  asm("{\n\t.reg .b32 lo, hi;\n\tmov.b64 {lo, hi}, %1;\n\t"
      "shfl.sync.up.b32 lo, lo, %2, 0, -1;\n\tshfl.sync.up.b32 hi, hi, %2, 0, -1;\n\t"
      "mov.b64 %0, {lo, hi};\n\t}"
      : "=d"(r)
      : "d"(x), "r"(d));
  return r;
}
__device__ __forceinline__ double shfl_idx_f64(double x, int src) {
  double r;
  asm("{\n\t.reg .b32 lo, hi;\n\tmov.b64 {lo, hi}, %1;\n\t"
      "shfl.sync.idx.b32 lo, lo, %2, 31, -1;\n\tshfl.sync.idx.b32 hi, hi, %2, 31, -1;\n\t"
      "mov.b64 %0, {lo, hi};\n\t}"
      : "=d"(r)
      : "d"(x), "r"(src));
  return r;
}
// s += P o (2 x 2, P column-major as two double2).
__device__ __forceinline__ void fma2(double& s0, double& s1, double2 p01, double2 p23, double o0, double o1) {
  s0 = fma(p23.x, o1, fma(p01.x, o0, s0));
  s1 = fma(p23.y, o1, fma(p01.y, o0, s1));
}

constexpr int kLineSmemBudget = 96 * 1024;  // bytes of trace lines per block kept in smem
constexpr int kWarps = 8;                   // warps per block
constexpr int kCpl = 2;                     // adjacent cells per lane
constexpr int kChunk = 32 * kCpl;           // cells per warp step
constexpr int kAheadChunks = 4;             // minimum L2 prefetch distance (chunks)

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

__device__ __forceinline__ void mat2_vec(const double* G, double x0, double x1, double& y0, double& y1) {
  y0 = G[0] * x0 + G[2] * x1;  // column-major 2 x 2
  y1 = G[1] * x0 + G[3] * x1;
}

// Warps per direction: kOne (one warp), kRows (warp w owns rows w, w+W, ...;
// reads warp w-1's trace line behind its progress counter) or kSplit (warp
// s owns column segment s of every row; its trace line covers only its
// segment, and the x-carry at the segment boundary comes from warp s-1
// through a per-row slot in global memory behind warp s-1's row counter).
enum SweepMode { kOne = 0, kRows = 1, kSplit = 2 };

// One warp's share of one direction.
struct Dir {
  const double* rhs;
  const double* bc;
  double* psi;
  const double* sigma_t;
  const double* cst;  // shared memory, kConsts
  int* prod;          // shared memory, W progress counters
  double* my_line;
  const double* in_line;
  double* carry;      // kSplit: (W-1) x ny x 2 boundary carries
  const double* pref;  // general media: this direction's prefactored block data (or nullptr)
  long long pref_stride;
  int* err;
  int nx, ny, W, w, pw, nchunk, nrows, pitch;
  int rw, rW;         // row interleave: rows rw, rw + rW, ... (kRows: w, W; else 0, 1)
  int kbeg, kend;     // this warp's chunk range within a row
  bool yu, smem_lines;
};

template <bool UNIFORM, int MODE, bool HAS_BC, bool XU>
__device__ __forceinline__ void sweep_dir(const Dir& d) {
  constexpr bool MULTI = MODE == kRows, SPLIT = MODE == kSplit;
  constexpr int kDx = XU ? 1 : -1;  // cell index step along the sweep
  const int lane = threadIdx.x & 31;
  const int nx = d.nx, nrows = d.nrows, kbeg = d.kbeg, kend = d.kend;
  const int nchunk = kend - kbeg;  // chunks per row of this warp
  const int colbase = kbeg * kChunk;  // first sweep column of this warp's segment
  const int c0 = kCpl * lane;  // this lane's first sweep column within a chunk
  const double kx0 = d.cst[kKT], kx1 = d.cst[kKT + 1], tx0 = d.cst[kKT + 2], tx1 = d.cst[kKT + 3];
  const double ky0 = d.cst[kKT + 4], ky1 = d.cst[kKT + 5], ty0 = d.cst[kKT + 6], ty1 = d.cst[kKT + 7];
  const double2* c2 = reinterpret_cast<const double2*>(d.cst);

  auto row0_of = [&](int rowk) -> long long {
    const int r = d.rw + rowk * d.rW;
    return static_cast<long long>(d.yu ? r : d.ny - 1 - r) * nx;
  };
  // this lane's first cell of the warp's segment in row ordinal rowk
  auto first_cell = [&](int rowk) -> long long {
    return row0_of(rowk) + (XU ? colbase + c0 : nx - 1 - colbase - c0);
  };

  // L2 prefetch, one chunk per step kAheadChunks ahead, issued by lane 0;
  // (prow, pk) walks the chunks in sweep order.
  int prow = 0, pk = kbeg;
  long long prow0 = row0_of(0);
  // (general media with prefactored blocks: lanes 1..28 prefetch the 28
  // structure-of-arrays planes of the same chunk; every lane then walks.)
  const bool pf_lane = UNIFORM ? lane == 0 : (lane == 0 || (d.pref && lane <= kPrefDoubles));
  auto prefetch_next = [&]() {
    if (prow >= nrows) return;
    const int lo = pk * kChunk, cnt = min(kChunk, nx - lo);
    const long long first = prow0 + (XU ? lo : nx - lo - cnt);
    if (lane == 0) {
      prefetch_l2(d.rhs + 4 * first, static_cast<unsigned>(cnt) * 32u);
      if (HAS_BC) prefetch_l2(d.bc + 4 * first, static_cast<unsigned>(cnt) * 32u);
    } else if (!UNIFORM) {
      prefetch_l2(d.pref + (lane - 1) * d.pref_stride + first, static_cast<unsigned>(cnt) * 8u);
    }
    if (++pk == kend) {
      pk = kbeg;
      if (++prow < nrows) prow0 = row0_of(prow);
    }
  };
  if (pf_lane)
    for (int u = 0; u < kAheadChunks; ++u) prefetch_next();

  const int nsteps = nrows * nchunk;
  long long cell = first_cell(0);  // this lane's first cell of the current step
  long long next_row = nrows > 1 ? first_cell(1) : 0;
  int rowk = 0, k = kbeg;
  double tc0 = 0.0, tc1 = 0.0;  // x-trace carry into the chunk (lane 0)

  double ra0[4], ra1[4], rb0[4], rb1[4];  // two register sets of sources
  if (colbase + c0 < nx) ld_cell256(d.rhs + 4 * cell, ra0);
  if (colbase + c0 + 1 < nx) ld_cell256(d.rhs + 4 * (cell + kDx), ra1);

  auto step = [&](int t, double (&v0)[4], double (&v1)[4], double (&n0)[4], double (&n1)[4]) {
    const int col = k * kChunk + c0;
    const bool act0 = col < nx, act1 = col + 1 < nx;
    // next step's sources into the other register set
    const bool last = k + 1 == kend;
    const long long ncell = last ? next_row : cell + kDx * kChunk;
    const int ncol = last ? colbase + c0 : col + kChunk;
    if (t + 1 < nsteps) {
      if (ncol < nx) ld_cell256(d.rhs + 4 * ncell, n0);
      if (ncol + 1 < nx) ld_cell256(d.rhs + 4 * (ncell + kDx), n1);
    }
    if (pf_lane) prefetch_next();
    if (k == kbeg) {  // x-inflow of the row (segment): vacuum, or warp s-1's boundary carry
      tc0 = tc1 = 0.0;
      if (SPLIT && d.w > 0) {
        if (lane == 0) {
          wait_progress(d.prod + d.w - 1, rowk + 1);
          const double2 cin = __ldcg(reinterpret_cast<const double2*>(d.carry) + (d.w - 1) * d.ny + rowk);
          tc0 = cin.x;
          tc1 = cin.y;
        }
        __syncwarp();  // reconverge after lane 0's spin, or every shuffle takes the divergent path
      }
    }
    if (HAS_BC) {
      double g0[4], g1[4];
      if (act0) ld_cell256(d.bc + 4 * cell, g0);
      if (act1) ld_cell256(d.bc + 4 * (cell + kDx), g1);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        v0[i] += act0 ? g0[i] : 0.0;
        v1[i] += act1 ? g1[i] : 0.0;
      }
    }
    // y-upwind traces (per x-mode) of these columns from the previous row
    double y00 = 0.0, y01 = 0.0, y10 = 0.0, y11 = 0.0;  // y{cell}{x-mode}
    if (d.rw + rowk * d.rW > 0) {
      if (MULTI) {
        if (lane == 0) wait_progress(d.prod + d.pw, (d.w == 0 ? rowk - 1 : rowk) * nchunk + k + 1);
        __syncwarp();
      }
      if (act0) {
        const double2 p0 = ld_line(d.in_line + (col - colbase), d.smem_lines);
        const double2 p1 = ld_line(d.in_line + d.pitch + (col - colbase), d.smem_lines);
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
      // f = T_x u (per y-mode); lane map over its two cells: tau -> G^2 tau + (G f0 + f1);
      // lane 0 also applies its map to the chunk's carry.
      const double f00 = tx0 * u0[0] + tx1 * u0[1], f01 = tx0 * u0[2] + tx1 * u0[3];
      const double f10 = tx0 * u1[0] + tx1 * u1[1], f11 = tx0 * u1[2] + tx1 * u1[3];
      const double2 g01 = c2[kG / 2], g23 = c2[kG / 2 + 1];
      double s0 = f10 + g01.x * f00 + g23.x * f01;
      double s1 = f11 + g01.y * f00 + g23.y * f01;
      fma2(s0, s1, c2[kGP / 2], c2[kGP / 2 + 1], tc0, tc1);  // tc = 0 off lane 0
      // inclusive scan over the lanes: s_l <- s_l + G^(2d) s_{l-d}
#pragma unroll
      for (int l = 0; l < 5; ++l) {
        const int dd = 1 << l;
        double o0 = shfl_up_f64(s0, dd);
        double o1 = shfl_up_f64(s1, dd);
        o0 = lane >= dd ? o0 : 0.0;
        o1 = lane >= dd ? o1 : 0.0;
        fma2(s0, s1, c2[(kGP + 4 * (dd - 1)) / 2], c2[(kGP + 4 * (dd - 1)) / 2 + 1], o0, o1);
      }
      // One rotation: lane l > 0 receives tau_in from lane l-1; lane 0
      // receives lane 31's tau, the next chunk's carry (only lane 0 keeps one).
      double ti0 = shfl_idx_f64(s0, (lane + 31) & 31);
      double ti1 = shfl_idx_f64(s1, (lane + 31) & 31);
      if (lane == 0) {
        const double n0 = ti0, n1 = ti1;
        ti0 = tc0, ti1 = tc1;
        tc0 = n0, tc1 = n1;
      }
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
      double Qc0[8], Qc1[8], G0[4], G1[4];
      if (d.pref) {
        // prefactored (launch_sweep_prefactor): M^-1, Qc and G of the lane's cell
        // pair, structure of arrays, the pair's lower cell first
        const long long lo = act0 ? (XU ? cell : cell + kDx) : 0;
        const double* tb = d.pref + lo;
        auto pair = [&](int k) { return __ldg(reinterpret_cast<const double2*>(tb + k * d.pref_stride)); };
        double u0[4] = {0.0, 0.0, 0.0, 0.0}, u1[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const double2 m = pair(c * 4 + i);
            u0[i] = fma(XU ? m.x : m.y, v0[c], u0[i]);
            u1[i] = fma(XU ? m.y : m.x, v1[c], u1[i]);
          }
#pragma unroll
        for (int i = 0; i < 4; ++i) v0[i] = u0[i], v1[i] = u1[i];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const double2 q = pair(16 + e);
          Qc0[e] = XU ? q.x : q.y;
          Qc1[e] = XU ? q.y : q.x;
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const double2 g = pair(24 + e);
          G0[e] = XU ? g.x : g.y;
          G1[e] = XU ? g.y : g.x;
        }
      } else {
      bool ok0, ok1;
      {
        double A[16];
        const double2* sb = reinterpret_cast<const double2*>(d.sigma_t + 16 * cell);
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
        const double2* sb = reinterpret_cast<const double2*>(d.sigma_t + 16 * (act1 ? cell + kDx : cell));
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
      if ((!ok0 && act0) || (!ok1 && act1)) atomicExch(d.err, 1);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        G0[c * 2 + 0] = tx0 * Qc0[c * 4 + 0] + tx1 * Qc0[c * 4 + 1];
        G0[c * 2 + 1] = tx0 * Qc0[c * 4 + 2] + tx1 * Qc0[c * 4 + 3];
        G1[c * 2 + 0] = tx0 * Qc1[c * 4 + 0] + tx1 * Qc1[c * 4 + 1];
        G1[c * 2 + 1] = tx0 * Qc1[c * 4 + 2] + tx1 * Qc1[c * 4 + 3];
      }
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
      fma2(s0, s1, make_double2(A0, A1), make_double2(A2, A3), tc0, tc1);  // the carry (0 off lane 0)
#pragma unroll
      for (int l = 0; l < 5; ++l) {
        const int dd = 1 << l;
        const bool in = lane >= dd;
        double p0 = shfl_up_f64(A0, dd), p1 = shfl_up_f64(A1, dd);
        double p2 = shfl_up_f64(A2, dd), p3 = shfl_up_f64(A3, dd);
        double o0 = shfl_up_f64(s0, dd), o1 = shfl_up_f64(s1, dd);
        p0 = in ? p0 : 1.0;  // identity map below lane dd
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
      double ti0 = shfl_idx_f64(s0, (lane + 31) & 31);
      double ti1 = shfl_idx_f64(s1, (lane + 31) & 31);
      if (lane == 0) {
        const double n0 = ti0, n1 = ti1;
        ti0 = tc0, ti1 = tc1;
        tc0 = n0, tc1 = n1;
      }
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
      double* p = d.psi + 4 * cell;
      st_cell256(p, ps0);
      if (act1) st_cell256(p + 4 * kDx, ps1);
      // y-outflow traces (per x-mode) for the next row
      st_line(d.my_line + (col - colbase), ty0 * ps0[0] + ty1 * ps0[2], ty0 * ps1[0] + ty1 * ps1[2],
              d.smem_lines);
      st_line(d.my_line + d.pitch + (col - colbase), ty0 * ps0[1] + ty1 * ps0[3], ty0 * ps1[1] + ty1 * ps1[3],
              d.smem_lines);
    }
    __syncwarp();  // (own line: the next row reads what this row wrote)
    if (MULTI && lane == 0) publish_progress(d.prod + d.w, t + 1);
    if (SPLIT && last && d.w + 1 < d.W) {
      // the carry out of this segment's last (full) chunk: lane 0 holds it after the rotation
      if (lane == 0) {
        __stcg(reinterpret_cast<double2*>(d.carry) + d.w * d.ny + rowk, make_double2(tc0, tc1));
        publish_progress(d.prod + d.w, rowk + 1);
      }
      __syncwarp();
    }
    // advance
    cell = ncell;
    if (last) {
      k = kbeg;
      ++rowk;
      next_row = rowk + 1 < nrows ? first_cell(rowk + 1) : 0;
    } else {
      ++k;
    }
  };

  for (int t = 0; t < nsteps; t += 2) {
    step(t, ra0, ra1, rb0, rb1);
    if (t + 1 < nsteps) step(t + 1, rb0, rb1, ra0, ra1);
  }
}

// nck: chunks per segment (kSplit); the trace lines then span one segment.
template <bool UNIFORM, int MODE, bool HAS_BC>
__global__ void __launch_bounds__(256, 2) sweep_scan_kernel(const SweepArgs a, int W, bool smem_lines, int nck) {
  extern __shared__ double smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int groups = kWarps / W;
  const int g = wib / W, w = wib % W;
  const int slot = blockIdx.x * groups + g;
  if (slot >= a.n) return;  // a whole direction group exits together
  const int nx = a.nx, ny = a.ny;
  const int linew = MODE == kSplit ? nck * kChunk : nx;  // columns per trace line
  const int pitch = line_pitch(linew);
  double* base = smem + static_cast<size_t>(g) * group_doubles(W, linew, smem_lines);
  double* cst = base;
  int* prod = reinterpret_cast<int*>(base + kConsts);
  double* lines = smem_lines ? base + kConsts + 2 * ((W + 3) / 4) : a.line + static_cast<size_t>(slot) * W * 2 * pitch;
  const int ang = a.angles ? a.angles[slot] : slot;
  const double omx = a.dirs[3 * ang], omy = a.dirs[3 * ang + 1];
  const bool xu = omx >= 0.0, yu = omy >= 0.0;  // sweep.cpp:37-38
  if (w == 0) {
    const double* ax = xu ? a.sc.ax_minus : a.sc.ax_plus;
    const double* ay = yu ? a.sc.ay_minus : a.sc.ay_plus;
    if (lane < 16) {
      const double dv = omx * ax[lane] + omy * ay[lane];
      cst[lane] = UNIFORM ? dv + a.sigma_t[lane] : dv;
    }
    if (lane < 2) {
      // (B psi_up)[my,mx] = c[mx] (t . psi_up[my,:]), (c,t) = (-t_L,t_R) minus / (t_R,t_L) plus
      cst[kKT + lane] = omx * (xu ? -a.sc.trx_l[lane] : a.sc.trx_r[lane]);
      cst[kKT + 2 + lane] = xu ? a.sc.trx_r[lane] : a.sc.trx_l[lane];
      cst[kKT + 4 + lane] = omy * (yu ? -a.sc.try_l[lane] : a.sc.try_r[lane]);
      cst[kKT + 6 + lane] = yu ? a.sc.try_r[lane] : a.sc.try_l[lane];
    }
    __syncwarp();
    if (UNIFORM && lane == 0) {
      // M^-1 columns via the reference LU; Q = -M^-1 K_x; G = T_x Q; (G^2)^(l+1)
      double Mi[16];
      for (int c = 0; c < 4; c += 3) {
        double A[16], e0[4] = {0, 0, 0, 0}, e1[4] = {0, 0, 0, 0}, e2[4] = {0, 0, 0, 0};
        for (int k = 0; k < 16; ++k) A[k] = cst[k];
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
      const double kx0 = cst[kKT], kx1 = cst[kKT + 1], tx0 = cst[kKT + 2], tx1 = cst[kKT + 3];
      // K_x (4 x 2): column my has kx[mx] at rows (my, mx)
      double Q[8];
      for (int my = 0; my < 2; ++my)
        for (int r = 0; r < 4; ++r)
          Q[my * 4 + r] = -(Mi[(my * 2 + 0) * 4 + r] * kx0 + Mi[(my * 2 + 1) * 4 + r] * kx1);
      // G = T_x Q (2 x 2): row m = tx . Q[(m,0..1), :]
      double Gm[4];
      for (int col = 0; col < 2; ++col)
        for (int m = 0; m < 2; ++m) Gm[col * 2 + m] = tx0 * Q[col * 4 + m * 2] + tx1 * Q[col * 4 + m * 2 + 1];
      for (int k = 0; k < 16; ++k) cst[k] = Mi[k];
      for (int k = 0; k < 8; ++k) cst[kQ + k] = Q[k];
      for (int e = 0; e < 4; ++e) cst[kG + e] = Gm[e];
      double G2[4];
      for (int col = 0; col < 2; ++col)
        for (int m = 0; m < 2; ++m) G2[col * 2 + m] = Gm[m] * Gm[col * 2] + Gm[2 + m] * Gm[col * 2 + 1];
      double P[4] = {G2[0], G2[1], G2[2], G2[3]};
      for (int k = 0; k < 32; ++k) {
        for (int e = 0; e < 4; ++e) cst[kGP + 4 * k + e] = P[e];
        double N[4];
        for (int col = 0; col < 2; ++col)
          for (int m = 0; m < 2; ++m) N[col * 2 + m] = G2[m] * P[col * 2] + G2[2 + m] * P[col * 2 + 1];
        for (int e = 0; e < 4; ++e) P[e] = N[e];
      }
    }
    if (lane < W) prod[lane] = 0;
  }
  asm volatile("bar.sync %0, %1;" ::"r"(g + 1), "r"(W * 32) : "memory");

  Dir d;
  d.rhs = a.rhs + static_cast<long long>(slot) * a.rhs_stride;
  d.bc = HAS_BC ? a.bc + static_cast<long long>(ang) * a.bc_stride : nullptr;
  d.psi = a.psi + static_cast<long long>(slot) * a.psi_stride;
  d.sigma_t = a.sigma_t;
  d.cst = cst;
  d.prod = prod;
  d.pw = (w + W - 1) % W;
  d.my_line = lines + static_cast<size_t>(w) * 2 * pitch;
  // kRows reads warp w-1's line (the previous row); otherwise a warp's own
  // line holds its columns of the previous row
  d.in_line = lines + static_cast<size_t>(MODE == kRows ? d.pw : w) * 2 * pitch;
  d.err = a.err;
  d.pref = a.pref ? a.pref + static_cast<long long>(slot) * kPrefDoubles * a.pref_stride : nullptr;
  d.pref_stride = a.pref_stride;
  d.nx = nx;
  d.ny = ny;
  d.W = W;
  d.w = w;
  d.nchunk = (nx + kChunk - 1) / kChunk;
  if (MODE == kSplit) {  // segment w of every row; boundary carries in the (unused) global line buffer
    d.rw = 0;
    d.rW = 1;
    d.nrows = ny;
    d.kbeg = w * nck;
    d.kend = min(d.nchunk, (w + 1) * nck);
    d.carry = a.line + static_cast<size_t>(slot) * (W - 1) * ny * 2;
  } else {
    d.rw = w;
    d.rW = W;
    d.nrows = (ny - w + W - 1) / W;  // rows w, w+W, ... of this warp
    d.kbeg = 0;
    d.kend = d.nchunk;
    d.carry = nullptr;
  }
  d.pitch = pitch;
  d.yu = yu;
  d.smem_lines = smem_lines;
  if (xu)
    sweep_dir<UNIFORM, MODE, HAS_BC, true>(d);
  else
    sweep_dir<UNIFORM, MODE, HAS_BC, false>(d);
}

// Per (direction slot, cell): the block M = Omega_x A_x + Omega_y A_y +
// Sigma_t(cell) in the sweep's own arithmetic, factored with the reference's
// partial-pivot LU (singular test as sweep.cpp:49-52), and written as M^-1,
// Qc = -M^-1 K_x and G = T_x Qc, structure of arrays.
__global__ void __launch_bounds__(256) sweep_prefactor_kernel(const SweepArgs a, double* __restrict__ table,
                                                              long long stride) {
  const int slot = blockIdx.y;
  const long long c = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  const long long ncell = static_cast<long long>(a.nx) * a.ny;
  if (c >= ncell) return;
  const int ang = a.angles ? a.angles[slot] : slot;
  const double omx = a.dirs[3 * ang], omy = a.dirs[3 * ang + 1];
  const bool xu = omx >= 0.0, yu = omy >= 0.0;
  const double* ax = xu ? a.sc.ax_minus : a.sc.ax_plus;
  const double* ay = yu ? a.sc.ay_minus : a.sc.ay_plus;
  double M[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) M[k] = (omx * ax[k] + omy * ay[k]) + a.sigma_t[16 * c + k];
  double Mi[16];
  bool ok = true;
#pragma unroll
  for (int c0 = 0; c0 < 4; c0 += 3) {
    double A[16], e0[4] = {0, 0, 0, 0}, e1[4] = {0, 0, 0, 0}, e2[4] = {0, 0, 0, 0};
#pragma unroll
    for (int k = 0; k < 16; ++k) A[k] = M[k];
    e0[c0] = 1.0;
    if (c0 + 1 < 4) e1[c0 + 1] = 1.0;
    if (c0 + 2 < 4) e2[c0 + 2] = 1.0;
    ok = lu_solve4x3(A, e0, e1, e2) && ok;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      Mi[c0 * 4 + r] = e0[r];
      if (c0 + 1 < 4) Mi[(c0 + 1) * 4 + r] = e1[r];
      if (c0 + 2 < 4) Mi[(c0 + 2) * 4 + r] = e2[r];
    }
  }
  if (!ok) atomicExch(a.err, 1);
  const double kx0 = omx * (xu ? -a.sc.trx_l[0] : a.sc.trx_r[0]), kx1 = omx * (xu ? -a.sc.trx_l[1] : a.sc.trx_r[1]);
  const double tx0 = xu ? a.sc.trx_r[0] : a.sc.trx_l[0], tx1 = xu ? a.sc.trx_r[1] : a.sc.trx_l[1];
  double* t = table + static_cast<long long>(slot) * kPrefDoubles * stride + c;
#pragma unroll
  for (int k = 0; k < 16; ++k) t[k * stride] = Mi[k];
  double Q[8];
#pragma unroll
  for (int my = 0; my < 2; ++my)
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      Q[my * 4 + r] = -(Mi[(my * 2 + 0) * 4 + r] * kx0 + Mi[(my * 2 + 1) * 4 + r] * kx1);
      t[(16 + my * 4 + r) * stride] = Q[my * 4 + r];
    }
#pragma unroll
  for (int col = 0; col < 2; ++col)
#pragma unroll
    for (int m = 0; m < 2; ++m) t[(24 + col * 2 + m) * stride] = tx0 * Q[col * 4 + m * 2] + tx1 * Q[col * 4 + m * 2 + 1];
}

int sm_count() {
  static const int n = [] {
    int dev = 0, v = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

}  // namespace

void launch_sweep_prefactor(const SweepArgs& a, double* table, long long stride, cudaStream_t s) {
  if (a.n <= 0) return;
  const long long ncell = static_cast<long long>(a.nx) * a.ny;
  sweep_prefactor_kernel<<<dim3(static_cast<unsigned>((ncell + 255) / 256), a.n), 256, 0, s>>>(a, table, stride);
  RTLR_CUDA(cudaGetLastError());
}

void launch_sweep_scan(const SweepArgs& a, bool uniform, cudaStream_t s) {
  if (a.n <= 0) return;
  const int nchunk = (a.nx + kChunk - 1) / kChunk;
  auto lines_fit = [](int linew) {
    return static_cast<size_t>(kWarps) * 2 * line_pitch(linew) * sizeof(double) <= kLineSmemBudget;
  };
  // Last-wave fill of n*c warps over the resident warp slots (SMs x blocks/SM x kWarps).
  auto wave_eff = [&](int c, int linew, bool smem_lines) {
    const size_t smem = static_cast<size_t>(kWarps / c) * group_doubles(c, linew, smem_lines) * sizeof(double);
    const int per_sm = std::max(1, std::min(2, static_cast<int>((227u * 1024u) / (smem + 1024u))));
    const double slots = static_cast<double>(sm_count()) * per_sm * kWarps;
    const double waves = static_cast<double>(a.n) * c / slots;
    return waves <= 1.0 ? waves : waves / std::ceil(waves);
  };
  // Warps per direction W in {1, 2, 4, 8}, best last-wave fill, ties keep the
  // smaller W.  Rows whose full-width trace lines fit shared memory (nx <=
  // 768): row interleave (at most one warp per 2 rows).  Wider rows: column
  // segments (every segment non-empty, lines of one segment in shared
  // memory); only if no split fits do the lines go to L2.
  int mode = kOne, W = 1, nck = nchunk, linew = a.nx;
  bool smem_lines = lines_fit(a.nx);
  double best = -1.0;
  if (smem_lines) {
    for (int c = 1; c <= kWarps && (c == 1 || 2 * c <= a.ny); c *= 2) {
      const double eff = wave_eff(c, a.nx, true);
      if (eff > best + 1e-3) best = eff, W = c;
    }
    mode = W > 1 ? kRows : kOne;
  } else {
    for (int c = 2; c <= kWarps; c *= 2) {
      const int k = (nchunk + c - 1) / c;
      if ((c - 1) * k >= nchunk || !lines_fit(k * kChunk)) continue;
      const double eff = wave_eff(c, k * kChunk, true);
      if (eff > best + 1e-3) best = eff, W = c, nck = k;
    }
    if (W > 1) {
      mode = kSplit;
      smem_lines = true;
      linew = nck * kChunk;
    } else {  // rows in L2
      for (int c = 1; c <= kWarps && (c == 1 || 2 * c <= a.ny); c *= 2) {
        const double eff = wave_eff(c, a.nx, false);
        if (eff > best + 1e-3) best = eff, W = c;
      }
      mode = W > 1 ? kRows : kOne;
    }
  }
  const int groups = kWarps / W;
  const int blocks = (a.n + groups - 1) / groups;
  const size_t smem = static_cast<size_t>(groups) * group_doubles(W, linew, smem_lines) * sizeof(double);
  auto go = [&](auto kern) {
    RTLR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    kern<<<blocks, kWarps * 32, smem, s>>>(a, W, smem_lines, nck);
  };
  const bool bc = a.bc != nullptr;
#define RTLR_SCAN_GO(U, M) (bc ? go(sweep_scan_kernel<U, M, true>) : go(sweep_scan_kernel<U, M, false>))
  if (uniform) {
    if (mode == kSplit) RTLR_SCAN_GO(true, kSplit);
    else if (mode == kRows) RTLR_SCAN_GO(true, kRows);
    else RTLR_SCAN_GO(true, kOne);
  } else {
    if (mode == kSplit) RTLR_SCAN_GO(false, kSplit);
    else if (mode == kRows) RTLR_SCAN_GO(false, kRows);
    else RTLR_SCAN_GO(false, kOne);
  }
#undef RTLR_SCAN_GO
  RTLR_CUDA(cudaGetLastError());
}

}  // namespace cuda
}  // namespace rtlr
