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
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <stdexcept>
#include <vector>

#include <cuda.h>  // CUtensorMap (the encoder is fetched through the runtime)

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

// mbarrier and TMA primitives (shared-memory addresses as 32-bit offsets).
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
// One 2-D tile (16 rows of 128 B) of the source tensor into shared memory,
// completing its bytes on bar.
__device__ __forceinline__ void tma_load_tile(unsigned dst, const CUtensorMap* map, unsigned bar, int row) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(map), "r"(bar), "r"(0), "r"(row)
      : "memory");
}
// One 4 KB tile (32 tensor rows of 128 B) from shared memory to the tensor,
// as a bulk-group store (the TMA engine reads the tile asynchronously).
__device__ __forceinline__ void tma_store_tile(const CUtensorMap* map, int row, unsigned src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(map), "r"(src),
               "r"(0), "r"(row)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void st_shared_v2(unsigned addr, double x, double y) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(addr), "d"(x), "d"(y) : "memory");
}
__device__ __forceinline__ void ld_shared_v2(unsigned addr, double& x, double& y) {
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(addr) : "memory");
}

constexpr int kLineSmemBudget = 96 * 1024;  // bytes of trace lines per block kept in smem
constexpr int kWarps = 8;                   // warps per block
constexpr int kCpl = 2;                     // adjacent cells per lane
constexpr int kChunk = 32 * kCpl;           // cells per warp step
constexpr int kAheadChunks = 4;             // minimum L2 prefetch distance (chunks)
// Wide uniform kernel (sweep_dir_wide): four adjacent cells per lane, 128-cell
// chunks, sources through a per-warp TMA ring of 4 KB tiles (32 rows of
// 128 B, 128-byte swizzle: the lanes' 16-byte reads are bank-conflict free).
constexpr int kWCpl = 4;
constexpr int kWChunk = 32 * kWCpl;
constexpr int kWTileBytes = kWChunk * 32;
constexpr int kMaxStages = 6;

// Per-direction constants (shared memory, written by warp 0 of the group):
//   [0..16)   M^-1 (uniform) or Omega_x Ax + Omega_y Ay (general), column-major
//   [16..24)  kx[2] tx[2] ky[2] ty[2]
//   [24..32)  Q = -M^-1 K_x (4 x 2, uniform)
//   [32..36)  G = T_x Q (2 x 2, uniform)
//   [36..164) G^(2(l+1)), l = 0..31 (uniform): the map of 2(l+1) cells
constexpr int kKT = 16, kQ = 24, kG = 32, kGP = 36, kConsts = 164;

// Doubles per trace plane (even, so both planes stay 16-byte aligned).
__host__ __device__ constexpr int line_pitch(int nx) { return (nx + 1) & ~1; }
// The wide kernel reads and writes four columns (32 B) per lane: its lines
// carry two doubles of padding after every 16 columns, so the 8 lanes of a
// 16-byte shared-memory phase hit distinct banks (unpadded, lanes l and l+4
// collide).
__host__ __device__ constexpr int wide_line_idx(int c) { return c + 2 * (c >> 4); }
__host__ __device__ constexpr int line_pitch_w(int nx, bool wide) {
  return wide ? (wide_line_idx((nx + 3) & ~3) + 3) & ~3 : line_pitch(nx);
}
__host__ __device__ constexpr int group_doubles(int W, int nx, bool smem_lines, bool wide = false) {
  return kConsts + 2 * ((W + 3) / 4) + (smem_lines ? W * 2 * line_pitch_w(nx, wide) : 0);
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
  const CUtensorMap* tmap;  // wide: the source tensor (rows of 128 B)
  unsigned ring, bars;      // wide: this warp's ring tiles and mbarriers (shared memory)
  long long src_row0;       // wide: first tensor row of this direction's sources
  int stages;               // wide: ring depth
  int stage_out;            // wide: psi through the consumed source tile: 1 coalesced read-back + stores, 2 TMA store
  const CUtensorMap* pmap;  // wide, stage_out == 2: the psi tensor (rows of 128 B)
  long long psi_row0;       // wide: first tensor row of this direction's psi
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

  // Uniform media: the per-direction constants live in registers for the
  // whole sweep (the kernel runs one block per SM for this).  Read from
  // shared memory every step they were ~half of the L1 data-pipe wavefronts,
  // the limiter once the power cap pulls the SM clock down.
  double2 creg[UNIFORM ? kConsts / 2 : 1];
  if (UNIFORM) {
#pragma unroll
    for (int i = 0; i < (UNIFORM ? kConsts / 2 : 1); ++i) creg[i] = c2[i];
  }
  auto C2 = [&](int i) -> double2 { return UNIFORM ? creg[UNIFORM ? i : 0] : c2[i]; };
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
        const double2 lo = C2(2 * c), hi = C2(2 * c + 1);
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
      const double2 g01 = C2(kG / 2), g23 = C2(kG / 2 + 1);
      double s0 = f10 + g01.x * f00 + g23.x * f01;
      double s1 = f11 + g01.y * f00 + g23.y * f01;
      fma2(s0, s1, C2(kGP / 2), C2(kGP / 2 + 1), tc0, tc1);  // tc = 0 off lane 0
      // inclusive scan over the lanes: s_l <- s_l + G^(2d) s_{l-d}
#pragma unroll
      for (int l = 0; l < 5; ++l) {
        const int dd = 1 << l;
        double o0 = shfl_up_f64(s0, dd);
        double o1 = shfl_up_f64(s1, dd);
        o0 = lane >= dd ? o0 : 0.0;
        o1 = lane >= dd ? o1 : 0.0;
        fma2(s0, s1, C2((kGP + 4 * (dd - 1)) / 2), C2((kGP + 4 * (dd - 1)) / 2 + 1), o0, o1);
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
        const double2 qa = C2(kQ / 2 + h), qb = C2(kQ / 2 + 2 + h);  // Q[2h..2h+1], Q[4+2h..]
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

// The uniform-medium sweep with four adjacent cells per lane (128-cell
// chunks): the per-direction constants live in registers, the sources
// arrive through a TMA ring (lane 0 keeps `stages` tiles in flight), and a
// lane composes its four cells' maps by Horner (tau -> G^4 tau + s), so the
// 5-level shuffle scan and the carry rotation are paid once per 128 cells.
// Trace lines are always in shared memory.  Same DAG, progress counters and
// column-split carries as sweep_dir.
template <int MODE, bool HAS_BC, bool XU>
__device__ __forceinline__ void sweep_dir_wide(const Dir& d) {
  constexpr bool MULTI = MODE == kRows, SPLIT = MODE == kSplit;
  constexpr int kDx = XU ? 1 : -1;
  constexpr int C = kWCpl;
  const int lane = threadIdx.x & 31;
  const int nx = d.nx, nrows = d.nrows, kbeg = d.kbeg, kend = d.kend;
  const int nchunk = kend - kbeg;
  const int colbase = kbeg * kWChunk;
  const int c0 = C * lane;
  const double* cs = d.cst;
  double Mi[16], Q[8], G[4], L[5][4];
#pragma unroll
  for (int k = 0; k < 16; ++k) Mi[k] = cs[k];
#pragma unroll
  for (int k = 0; k < 8; ++k) Q[k] = cs[kQ + k];
#pragma unroll
  for (int k = 0; k < 4; ++k) G[k] = cs[kG + k];
#pragma unroll
  for (int l = 0; l < 5; ++l)  // G^(4 d), d = 2^l: entry 2d - 1 of the G^(2(i+1)) table
#pragma unroll
    for (int k = 0; k < 4; ++k) L[l][k] = cs[kGP + 4 * ((2 << l) - 1) + k];
  const double tx0 = cs[kKT + 2], tx1 = cs[kKT + 3];
  const double ky0 = cs[kKT + 4], ky1 = cs[kKT + 5], ty0 = cs[kKT + 6], ty1 = cs[kKT + 7];

  auto row0_of = [&](int rowk) -> long long {
    const int r = d.rw + rowk * d.rW;
    return static_cast<long long>(d.yu ? r : d.ny - 1 - r) * nx;
  };
  auto first_cell = [&](int rowk) -> long long {
    return row0_of(rowk) + (XU ? colbase + c0 : nx - 1 - colbase - c0);
  };
  const int nsteps = nrows * nchunk;
  const int S = d.stages;

  // TMA producer (lane 0): (trow, tk) walks the chunks in sweep order; a
  // tile starts at its chunk's first cell in memory order (the box may run
  // past the row; rows past the tensor are zero-filled).  With inflow data
  // the chunk's bc cells are prefetched into L2 alongside.
  int tissued = 0, trow = 0, tk = kbeg, ist = 0;
  long long trow0 = row0_of(0);
  auto tma_issue = [&]() {
    if (tissued >= nsteps) return;
    const int lo = tk * kWChunk;
    const long long first = trow0 + (XU ? lo : nx - lo - kWChunk);  // multiple of 4 cells
    const unsigned bar = d.bars + 8u * ist;
    mbar_expect(bar, kWTileBytes);
    tma_load_tile(d.ring + ist * kWTileBytes, d.tmap, bar, static_cast<int>(d.src_row0 + first / 4));
    if (HAS_BC) {
      const int cnt = min(kWChunk, nx - lo);
      prefetch_l2(d.bc + 4 * (trow0 + (XU ? lo : nx - lo - cnt)), static_cast<unsigned>(cnt) * 32u);
    }
    if (++ist == S) ist = 0;
    ++tissued;
    if (++tk == kend) {
      tk = kbeg;
      if (++trow < nrows) trow0 = row0_of(trow);
    }
  };
  // (TMA-store mode refills a slot one step after it was consumed, once the
  // store that reads it has let go of it)
  const bool tst = d.stage_out == 2;
  bool owe = false;
  if (lane == 0)
    for (int u = 0; u < S; ++u) tma_issue();
  // this lane's cells in a tile: memory index m -> 128-B row m / 4 (the same
  // row for all four: XU ? lane : 31 - lane), 16-B unit 2 (m % 4) + h,
  // swizzled by the row (CU_TENSOR_MAP_SWIZZLE_128B)
  const int trw = XU ? lane : 31 - lane;
  const unsigned tbase = static_cast<unsigned>(trw * 128), tsw = static_cast<unsigned>(trw & 7);
  auto unit = [&](int c, int h) -> unsigned {
    const unsigned u = static_cast<unsigned>(2 * (XU ? c : 3 - c) + h);
    return tbase + ((u ^ tsw) << 4);
  };

  long long cell = first_cell(0);
  long long next_row = nrows > 1 ? first_cell(1) : 0;
  int rowk = 0, k = kbeg, st = 0;
  unsigned ph = 0;
  double tc0 = 0.0, tc1 = 0.0;  // x-trace carry into the chunk (lane 0)

  for (int t = 0; t < nsteps; ++t) {
    const int col = k * kWChunk + c0;
    bool act[C];
#pragma unroll
    for (int c = 0; c < C; ++c) act[c] = col + c < nx;
    const bool last = k + 1 == kend;
    double v[C][4];
    {
      mbar_wait(d.bars + 8u * st, ph);
      const unsigned tile = d.ring + st * kWTileBytes;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        ld_shared_v2(tile + unit(c, 0), v[c][0], v[c][1]);
        ld_shared_v2(tile + unit(c, 1), v[c][2], v[c][3]);
      }
    }
    if (k == kbeg) {  // x-inflow of the row (segment): vacuum, or warp s-1's boundary carry
      tc0 = tc1 = 0.0;
      if (SPLIT && d.w > 0) {
        if (lane == 0) {
          wait_progress(d.prod + d.w - 1, rowk + 1);
          const double2 cin = __ldcg(reinterpret_cast<const double2*>(d.carry) + (d.w - 1) * d.ny + rowk);
          tc0 = cin.x;
          tc1 = cin.y;
        }
        __syncwarp();
      }
    }
    if (HAS_BC) {
#pragma unroll
      for (int c = 0; c < C; ++c) {
        double g[4];
        if (act[c]) {
          ld_cell256(d.bc + 4 * (cell + kDx * c), g);
#pragma unroll
          for (int i = 0; i < 4; ++i) v[c][i] += g[i];
        }
      }
    }
    // y-upwind traces (per x-mode) of these columns from the previous row
    double y[C][2];
#pragma unroll
    for (int c = 0; c < C; ++c) y[c][0] = y[c][1] = 0.0;
    if (d.rw + rowk * d.rW > 0) {
      if (MULTI) {
        if (lane == 0) wait_progress(d.prod + d.pw, (d.w == 0 ? rowk - 1 : rowk) * nchunk + k + 1);
        __syncwarp();
      }
      if (act[0]) {
        const double* p0 = d.in_line + wide_line_idx(col - colbase);
#pragma unroll
        for (int pl = 0; pl < 2; ++pl) {
          const unsigned a0 = smem_u32(p0 + pl * d.pitch);
          ld_shared_v2(a0, y[0][pl], y[1][pl]);
          ld_shared_v2(a0 + 16u, y[2][pl], y[3][pl]);
        }
#pragma unroll
        for (int c = 1; c < C; ++c)  // columns past the row end hold stale values
          if (!act[c]) y[c][0] = y[c][1] = 0.0;
      }
    }
    // u = M^-1 (rhs - Omega_y By psi_y); f = T_x u (per y-mode)
    double u[C][4], f[C][2];
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const double w0 = v[c][0] - ky0 * y[c][0], w1 = v[c][1] - ky0 * y[c][1];
      const double w2 = v[c][2] - ky1 * y[c][0], w3 = v[c][3] - ky1 * y[c][1];
#pragma unroll
      for (int i = 0; i < 4; ++i) u[c][i] = Mi[i] * w0 + Mi[4 + i] * w1 + Mi[8 + i] * w2 + Mi[12 + i] * w3;
      f[c][0] = tx0 * u[c][0] + tx1 * u[c][1];
      f[c][1] = tx0 * u[c][2] + tx1 * u[c][3];
    }
    // lane map tau -> G^4 tau + s (Horner over the four cells); lane 0 also
    // applies it to the chunk's carry
    double s0 = f[0][0], s1 = f[0][1];
#pragma unroll
    for (int c = 1; c < C; ++c) {
      const double n0 = f[c][0] + G[0] * s0 + G[2] * s1;
      const double n1 = f[c][1] + G[1] * s0 + G[3] * s1;
      s0 = n0;
      s1 = n1;
    }
    fma2(s0, s1, make_double2(L[0][0], L[0][1]), make_double2(L[0][2], L[0][3]), tc0, tc1);  // tc = 0 off lane 0
#pragma unroll
    for (int l = 0; l < 5; ++l) {
      const int dd = 1 << l;
      double o0 = shfl_up_f64(s0, dd);
      double o1 = shfl_up_f64(s1, dd);
      o0 = lane >= dd ? o0 : 0.0;
      o1 = lane >= dd ? o1 : 0.0;
      fma2(s0, s1, make_double2(L[l][0], L[l][1]), make_double2(L[l][2], L[l][3]), o0, o1);
    }
    double ti0 = shfl_idx_f64(s0, (lane + 31) & 31);
    double ti1 = shfl_idx_f64(s1, (lane + 31) & 31);
    if (lane == 0) {
      const double n0 = ti0, n1 = ti1;
      ti0 = tc0, ti1 = tc1;
      tc0 = n0, tc1 = n1;
    }
    // psi_c = u_c + Q tau, tau <- G tau + f_c, cell by cell
    double ps[C][4];
#pragma unroll
    for (int c = 0; c < C; ++c) {
#pragma unroll
      for (int i = 0; i < 4; ++i) ps[c][i] = u[c][i] + Q[i] * ti0 + Q[4 + i] * ti1;
      if (c + 1 < C) {
        const double n0 = f[c][0] + G[0] * ti0 + G[2] * ti1;
        const double n1 = f[c][1] + G[1] * ti0 + G[3] * ti1;
        ti0 = n0;
        ti1 = n1;
      }
    }
    const bool full_chunk = (k + 1) * kWChunk <= nx;
    if (d.stage_out) {
      // psi through the consumed source tile: the lanes write their four
      // cells where they read the sources (swizzled, conflict free), then
      // store instruction q takes memory-order cells 32 q + lane, 1 KB
      // contiguous per instruction instead of 32-byte pieces 128 B apart
      // (ncu: 52 L1 wavefronts per store instruction, two thirds of the
      // kernel's L1 data-pipe load, against 8 + the staging's 16).
      const unsigned tile = d.ring + st * kWTileBytes;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        st_shared_v2(tile + unit(c, 0), ps[c][0], ps[c][1]);
        st_shared_v2(tile + unit(c, 1), ps[c][2], ps[c][3]);
      }
      if (tst) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the writers' side of the TMA store
      __syncwarp();
      const long long gstart = XU ? cell - c0 : cell + c0 - (kWChunk - 1);  // the chunk's first cell in memory
      if (tst && full_chunk) {
        // a whole chunk: one TMA store of the tile (no read-back, no store
        // instructions of the lanes); the engine un-swizzles it
        if (lane == 0) tma_store_tile(d.pmap, static_cast<int>(d.psi_row0 + gstart / 4), tile);
      } else {
      const unsigned rsw = static_cast<unsigned>((lane >> 2) & 7);
      const unsigned lb0 = static_cast<unsigned>((lane >> 2) * 128) + (((2u * (lane & 3)) ^ rsw) << 4);
      const unsigned lb1 = static_cast<unsigned>((lane >> 2) * 128) + (((2u * (lane & 3) + 1u) ^ rsw) << 4);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int m = 32 * q + lane;  // memory-order cell of the tile
        double o[4];
        ld_shared_v2(tile + 1024u * q + lb0, o[0], o[1]);
        ld_shared_v2(tile + 1024u * q + lb1, o[2], o[3]);
        const int j = XU ? m : kWChunk - 1 - m;  // its sweep-order column within the chunk
        if (k * kWChunk + j < nx) st_cell256(d.psi + 4 * (gstart + m), o);
      }
      }
    } else {
#pragma unroll
      for (int c = 0; c < C; ++c)
        if (act[c]) st_cell256(d.psi + 4 * (cell + kDx * c), ps[c]);
    }
    if (act[0]) {  // y-outflow traces (per x-mode) for the next row
      double* q0 = d.my_line + wide_line_idx(col - colbase);
#pragma unroll
      for (int pl = 0; pl < 2; ++pl) {
        double o[C];
#pragma unroll
        for (int c = 0; c < C; ++c) o[c] = ty0 * ps[c][pl] + ty1 * ps[c][2 + pl];
        st_line(q0 + pl * d.pitch, o[0], o[1], true);
        st_line(q0 + pl * d.pitch + 2, o[2], o[3], true);
      }
    }
    __syncwarp();  // (own line: the next row reads what this row wrote; the tile is consumed)
    if (lane == 0) {
      if (tst) {
        // refill the previous step's slot once its store has read it (the
        // newest store may still be reading this step's slot)
        if (owe) {
          if (full_chunk)
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          else  // (no store was issued this step: the newest group is the previous slot's)
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          tma_issue();
        }
        owe = true;
      } else {
        // (the staged psi was written to the tile through the generic proxy:
        // ordered before the TMA engine's refill of it)
        if (d.stage_out) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        tma_issue();  // refill the stage this step consumed
      }
    }
    if (++st == S) st = 0, ph ^= 1u;
    if (MULTI && lane == 0) publish_progress(d.prod + d.w, t + 1);
    if (SPLIT && last && d.w + 1 < d.W) {
      if (lane == 0) {
        __stcg(reinterpret_cast<double2*>(d.carry) + d.w * d.ny + rowk, make_double2(tc0, tc1));
        publish_progress(d.prod + d.w, rowk + 1);
      }
      __syncwarp();
    }
    if (last) {
      cell = next_row;
      k = kbeg;
      ++rowk;
      next_row = rowk + 1 < nrows ? first_cell(rowk + 1) : 0;
    } else {
      cell += kDx * kWChunk;
      ++k;
    }
  }
  if (tst && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // the tiles stay until read
}

// Per-direction constants (kConsts layout above), written by one warp.
template <bool UNIFORM>
__device__ __forceinline__ void dir_consts(const SweepArgs& a, double omx, double omy, bool xu, bool yu, double* cst,
                                           int lane) {
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
}

// nck: chunks per segment (kSplit); the trace lines then span one segment.
// WIDE (uniform media only): sweep_dir_wide with the TMA source ring of
// `stages` 4 KB tiles per warp at the front of dynamic shared memory.
template <bool UNIFORM, int MODE, bool HAS_BC, bool WIDE>
__global__ void __launch_bounds__(256, UNIFORM ? 1 : 2)
    sweep_scan_kernel(const SweepArgs a, int W, bool smem_lines, int nck, int stages,
                      const __grid_constant__ CUtensorMap tmap, const __grid_constant__ CUtensorMap pmap) {
  static_assert(!WIDE || UNIFORM, "the wide kernel is for uniform media");
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ __align__(8) unsigned long long tma_bars[WIDE ? kWarps * kMaxStages : 1];
  // ring tiles first (1024-byte aligned for the swizzle), then the groups
  const unsigned raw = smem_u32(smem_raw);
  const unsigned ring = (raw + 1023u) & ~1023u;
  double* smem =
      reinterpret_cast<double*>(smem_raw + (WIDE ? ring - raw + static_cast<unsigned>(kWarps * stages * kWTileBytes) : 0));
  constexpr int kCh = WIDE ? kWChunk : kChunk;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int groups = kWarps / W;
  const int g = wib / W, w = wib % W;
  const int slot = blockIdx.x * groups + g;
  if (slot >= a.n) return;  // a whole direction group exits together
  const int nx = a.nx, ny = a.ny;
  const int linew = MODE == kSplit ? nck * kCh : nx;  // columns per trace line
  const int pitch = line_pitch_w(linew, WIDE);
  double* base = smem + static_cast<size_t>(g) * group_doubles(W, linew, smem_lines, WIDE);
  double* cst = base;
  int* prod = reinterpret_cast<int*>(base + kConsts);
  double* lines = smem_lines ? base + kConsts + 2 * ((W + 3) / 4) : a.line + static_cast<size_t>(slot) * W * 2 * pitch;
  const int ang = a.angles ? a.angles[slot] : slot;
  const double omx = a.dirs[3 * ang], omy = a.dirs[3 * ang + 1];
  const bool xu = omx >= 0.0, yu = omy >= 0.0;  // sweep.cpp:37-38
  if (w == 0) {
    dir_consts<UNIFORM>(a, omx, omy, xu, yu, cst, lane);
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
  d.tmap = &tmap;
  d.ring = ring + static_cast<unsigned>(wib * stages * kWTileBytes);
  d.bars = smem_u32(tma_bars) + (WIDE ? 8u * kMaxStages * wib : 0u);
  d.src_row0 = static_cast<long long>(slot) * a.rhs_stride / 16;
  d.stages = stages;
  d.stage_out = a.stage_out;
  d.pmap = &pmap;
  d.psi_row0 = static_cast<long long>(slot) * a.psi_stride / 16;
  if (WIDE) {
    if (lane == 0) {
      for (int u = 0; u < stages; ++u) mbar_init(d.bars + 8u * u, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
  }
  d.pref = a.pref ? a.pref + static_cast<long long>(slot) * kPrefDoubles * a.pref_stride : nullptr;
  d.pref_stride = a.pref_stride;
  d.nx = nx;
  d.ny = ny;
  d.W = W;
  d.w = w;
  d.nchunk = (nx + kCh - 1) / kCh;
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
  if constexpr (WIDE) {
    if (xu)
      sweep_dir_wide<MODE, HAS_BC, true>(d);
    else
      sweep_dir_wide<MODE, HAS_BC, false>(d);
  } else {
    if (xu)
      sweep_dir<UNIFORM, MODE, HAS_BC, true>(d);
    else
      sweep_dir<UNIFORM, MODE, HAS_BC, false>(d);
  }
}

// Per (direction slot, cell): the block M = Omega_x A_x + Omega_y A_y +
// Sigma_t(cell) in the sweep's own arithmetic, factored with the reference's
// partial-pivot LU (singular test as sweep.cpp:49-52), and written as M^-1,
// Qc = -M^-1 K_x and G = T_x Qc, structure of arrays.
__global__ void __launch_bounds__(256) sweep_prefactor_kernel(const SweepArgs a, double* __restrict__ table,
                                                              long long stride, int planes) {
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
  double* t = table + static_cast<long long>(slot) * planes * stride + c;
#pragma unroll
  for (int k = 0; k < 16; ++k) t[k * stride] = Mi[k];
  if (planes == kPrefMinvDoubles) return;  // the wavefront kernel forms Qc and G itself
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

// ---------------------------------------------------------------- wavefront mode
// A few directions (the low-rank inner loop's p sampled directions) leave
// the row-chunk kernel latency-bound: one SM per direction, every chunk step
// (loads, LU-free block algebra, the scan) on the sweep DAG's critical path.
// Here one direction runs on a thread-block cluster of CS CTAs x 8 warps;
// global warp g (= rank*8 + warp) owns rows g, g + 8 CS, ...  Each 32-cell
// chunk step is split: everything independent of the upwind row (the source
// and block loads, u = M^-1 rhs, the y-coupling Qy = -M^-1 K_y, the scan's
// transfer-matrix products level by level) runs before the wait; after the
// previous row's traces arrive only the 2-vector scan, the carry and psi
// remain.  The y-outflow traces go straight into the next row's warp's
// shared memory (st.async into distributed shared memory, possibly another
// CTA of the cluster), completing bytes on that warp's per-chunk mbarrier.
constexpr int kWaveWarps = 8;
constexpr size_t kWaveSmemMax = 220 * 1024;

__device__ __forceinline__ unsigned cluster_ctarank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned map_cluster(unsigned saddr, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Row hand-off: the producer lanes push their y-outflow traces into the
// consumer warp's shared memory with st.async, each completing 16 bytes of
// transaction count on the consumer's per-chunk mbarrier; the consumer arms
// the barrier with the chunk's byte count and waits on its phase parity.  No
// fences on either side, and the wait is a hardware barrier test rather
// than a polled flag.
__device__ __forceinline__ void st_async_v2(unsigned addr, double x, double y, unsigned mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(addr),
               "d"(x), "d"(y), "r"(mbar)
               : "memory");
}
__device__ __forceinline__ void prefetch_line_l2(const double* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
__device__ __forceinline__ double shfl_i(double x, int src) { return shfl_idx_f64(x, src); }
// 2 x 2 column-major products
__device__ __forceinline__ void mm2(const double* A, const double* B, double* C) {
  C[0] = A[0] * B[0] + A[2] * B[1];
  C[1] = A[1] * B[0] + A[3] * B[1];
  C[2] = A[0] * B[2] + A[2] * B[3];
  C[3] = A[1] * B[2] + A[3] * B[3];
}

template <bool UNIFORM, bool HAS_BC>
__global__ void __launch_bounds__(256, 1) sweep_wave_kernel(const SweepArgs a, int CS) {
  extern __shared__ double smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const unsigned crank = cluster_ctarank();
  const int slot = blockIdx.x / CS;
  const int nx = a.nx, ny = a.ny;
  const int nchunk = (nx + 31) / 32;
  double* cst = smem;
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem + kConsts);  // kWaveWarps x nchunk
  double* lines = smem + kConsts + kWaveWarps * nchunk;  // kWaveWarps x nx x (mode 0, mode 1)
  const int ang = a.angles ? a.angles[slot] : slot;
  const double omx = a.dirs[3 * ang], omy = a.dirs[3 * ang + 1];
  const bool xu = omx >= 0.0, yu = omy >= 0.0;  // sweep.cpp:37-38
  if (wib == 0) dir_consts<UNIFORM>(a, omx, omy, xu, yu, cst, lane);
  for (int i = threadIdx.x; i < kWaveWarps * nchunk; i += blockDim.x) mbar_init(smem_u32(bars + i), 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  cluster_barrier();  // constants and initialised barriers before any remote store

  const int WT = CS * kWaveWarps;
  const int g = static_cast<int>(crank) * kWaveWarps + wib;
  const int gc = (g + 1) % WT;  // the warp owning the next row
  const unsigned out_line = map_cluster(smem_u32(lines + static_cast<size_t>(gc % kWaveWarps) * 2 * nx),
                                        static_cast<unsigned>(gc / kWaveWarps));
  const unsigned out_bar = map_cluster(smem_u32(bars + static_cast<size_t>(gc % kWaveWarps) * nchunk),
                                       static_cast<unsigned>(gc / kWaveWarps));
  const unsigned my_bar = smem_u32(bars + static_cast<size_t>(wib) * nchunk);
  const double* in_line = lines + static_cast<size_t>(wib) * 2 * nx;
  const double* rhs = a.rhs + static_cast<long long>(slot) * a.rhs_stride;
  const double* bc = HAS_BC ? a.bc + static_cast<long long>(ang) * a.bc_stride : nullptr;
  double* psi = a.psi + static_cast<long long>(slot) * a.psi_stride;
  const double* tb = UNIFORM ? nullptr : a.pref + static_cast<long long>(slot) * kPrefMinvDoubles * a.pref_stride;
  const long long ps = a.pref_stride;
  const double kx0 = cst[kKT], kx1 = cst[kKT + 1];
  const double tx0 = cst[kKT + 2], tx1 = cst[kKT + 3];
  const double ky0 = cst[kKT + 4], ky1 = cst[kKT + 5], ty0 = cst[kKT + 6], ty1 = cst[kKT + 7];
  auto cell_of = [&](int r, int col) -> long long {
    return static_cast<long long>(yu ? r : ny - 1 - r) * nx + (xu ? col : nx - 1 - col);
  };
  // L2 prefetch of the next chunk step's sources and block planes: 8 + 56
  // lines of 128 B, two per lane (per-lane prefetches: no uniform-address loop)
  auto prefetch = [&](int r, int k) {
    if (r >= ny) return;
    const int lo = k * 32, cnt = min(32, nx - lo);
    const long long first = static_cast<long long>(yu ? r : ny - 1 - r) * nx + (xu ? lo : nx - lo - cnt);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int i = lane + 32 * h;
      if (i < 8) {
        if (16 * i < 4 * cnt) prefetch_line_l2(rhs + 4 * first + 16 * i);
      } else if (!UNIFORM && i < 8 + 2 * kPrefMinvDoubles) {
        const int pl = (i - 8) >> 1, half = (i - 8) & 1;
        if (16 * half < cnt) prefetch_line_l2(tb + pl * ps + first + 16 * half);
      }
    }
    if (HAS_BC && lane < 8 && 16 * lane < 4 * cnt) prefetch_line_l2(bc + 4 * first + 16 * lane);
  };

  // Node q = (row ordinal j, chunk k) of this warp, row r = g + j WT.  The
  // sources and block planes of node q + 1 load into registers before node
  // q waits on its upwind row, so their latency hides behind the wait.
  const int nrow_w = g < ny ? (ny - g + WT - 1) / WT : 0;
  const int nodes = nrow_w * nchunk;
  auto node_cell = [&](int q) -> long long {
    const int col = (q % nchunk) * 32 + lane;
    return cell_of(g + (q / nchunk) * WT, col < nx ? col : nx - 1);
  };
  double dv[4], dt[UNIFORM ? 1 : kPrefMinvDoubles];
  auto load = [&](int q) {
    const long long c = node_cell(q);
    ld_cell256(rhs + 4 * c, dv);
    if (HAS_BC) {
      double gb[4];
      ld_cell256(bc + 4 * c, gb);
#pragma unroll
      for (int i = 0; i < 4; ++i) dv[i] += gb[i];
    }
    if (!UNIFORM) {
#pragma unroll
      for (int e = 0; e < kPrefMinvDoubles; ++e) dt[e] = __ldg(tb + c + e * ps);
    }
  };
  if (nodes > 0) load(0);
  double tc0 = 0.0, tc1 = 0.0;  // x-inflow of the chunk (every lane holds it)
  for (int q = 0; q < nodes; ++q) {
    const int j = q / nchunk, k = q - j * nchunk, r = g + j * WT;
    if (k == 0) tc0 = tc1 = 0.0;
    const unsigned parity = static_cast<unsigned>(g == 0 ? j - 1 : j) & 1u;  // this row's phase of the barriers
    {
      const unsigned bytes = 16u * static_cast<unsigned>(min(32, nx - 32 * k));
      if (r > 0 && lane == 0) mbar_expect(my_bar + 8u * k, bytes);
      if (q + 2 < nodes) {
        const int q2 = q + 2, j2 = q2 / nchunk;
        prefetch(g + j2 * WT, q2 - j2 * nchunk);
      }
      const int col = k * 32 + lane;
      const bool act = col < nx;
      const long long cell = cell_of(r, act ? col : nx - 1);
      // ---- independent of the upwind row
      double v[4] = {dv[0], dv[1], dv[2], dv[3]};
      double Mi[16], Qc[8], G[4];
      if (UNIFORM) {
#pragma unroll
        for (int e = 0; e < 16; ++e) Mi[e] = cst[e];
#pragma unroll
        for (int e = 0; e < 8; ++e) Qc[e] = cst[kQ + e];
#pragma unroll
        for (int e = 0; e < 4; ++e) G[e] = cst[kG + e];
      } else {
#pragma unroll
        for (int e = 0; e < 16; ++e) Mi[e] = dt[e];
        // Qc = -M^-1 K_x, G = T_x Qc (as sweep_prefactor_kernel)
#pragma unroll
        for (int my = 0; my < 2; ++my)
#pragma unroll
          for (int i = 0; i < 4; ++i) Qc[my * 4 + i] = -(Mi[(my * 2 + 0) * 4 + i] * kx0 + Mi[(my * 2 + 1) * 4 + i] * kx1);
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int m = 0; m < 2; ++m) G[c * 2 + m] = tx0 * Qc[c * 4 + m * 2] + tx1 * Qc[c * 4 + m * 2 + 1];
      }
      // u = M^-1 rhs; Qy = -M^-1 K_y (K_y: column mx has ky[my] at rows (my, mx))
      double u[4], Qy[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        u[i] = Mi[i] * v[0] + Mi[4 + i] * v[1] + Mi[8 + i] * v[2] + Mi[12 + i] * v[3];
        Qy[i] = -(ky0 * Mi[i] + ky1 * Mi[8 + i]);
        Qy[4 + i] = -(ky0 * Mi[4 + i] + ky1 * Mi[12 + i]);
      }
      // f = T_x u + Gy y, Gy = T_x Qy (rows: y-mode)
      double f0 = tx0 * u[0] + tx1 * u[1], f1 = tx0 * u[2] + tx1 * u[3];
      double Gy[4] = {tx0 * Qy[0] + tx1 * Qy[1], tx0 * Qy[2] + tx1 * Qy[3], tx0 * Qy[4] + tx1 * Qy[5],
                      tx0 * Qy[6] + tx1 * Qy[7]};
      if (q + 1 < nodes) load(q + 1);  // (v and the planes are consumed)
      if (!act) {  // past the row end (last in sweep order): the zero map
        f0 = f1 = 0.0;
#pragma unroll
        for (int e = 0; e < 4; ++e) G[e] = Gy[e] = 0.0;
      }
      // transfer-matrix scan: A_l before each level, the lane's prefix map after
      double Al[5][4], A[4] = {G[0], G[1], G[2], G[3]};
#pragma unroll
      for (int l = 0; l < 5; ++l) {
        const int dd = 1 << l;
        const bool in = lane >= dd;
#pragma unroll
        for (int e = 0; e < 4; ++e) Al[l][e] = A[e];
        double P[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) P[e] = shfl_up_f64(A[e], dd);
        if (!in) P[0] = 1.0, P[1] = 0.0, P[2] = 0.0, P[3] = 1.0;
        double N[4];
        mm2(A, P, N);
#pragma unroll
        for (int e = 0; e < 4; ++e) A[e] = N[e];
      }
      const int src = (lane + 31) & 31;
      double rA[4], A31[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        rA[e] = shfl_i(A[e], src);
        A31[e] = shfl_i(A[e], 31);
      }
      if (lane == 0) rA[0] = 1.0, rA[1] = 0.0, rA[2] = 0.0, rA[3] = 1.0;
      // ---- the previous row's traces
      double y0 = 0.0, y1 = 0.0;
      if (r > 0) {
        mbar_wait(my_bar + 8u * k, parity);
        if (act) {
          const double2 t2 = ld_line(in_line + 2 * col, true);
          y0 = t2.x;
          y1 = t2.y;
        }
      }
      // ---- dependent part
      double s0 = f0 + Gy[0] * y0 + Gy[2] * y1, s1 = f1 + Gy[1] * y0 + Gy[3] * y1;
#pragma unroll
      for (int l = 0; l < 5; ++l) {
        const int dd = 1 << l;
        double o0 = shfl_up_f64(s0, dd), o1 = shfl_up_f64(s1, dd);
        o0 = lane >= dd ? o0 : 0.0;
        o1 = lane >= dd ? o1 : 0.0;
        s0 += Al[l][0] * o0 + Al[l][2] * o1;
        s1 += Al[l][1] * o0 + Al[l][3] * o1;
      }
      double rs0 = shfl_i(s0, src), rs1 = shfl_i(s1, src);
      const double e0 = shfl_i(s0, 31), e1 = shfl_i(s1, 31);
      if (lane == 0) rs0 = rs1 = 0.0;
      const double ti0 = rs0 + rA[0] * tc0 + rA[2] * tc1, ti1 = rs1 + rA[1] * tc0 + rA[3] * tc1;
      const double n0 = e0 + A31[0] * tc0 + A31[2] * tc1, n1 = e1 + A31[1] * tc0 + A31[3] * tc1;
      tc0 = n0;
      tc1 = n1;
      double p[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) p[i] = u[i] + Qy[i] * y0 + Qy[4 + i] * y1 + Qc[i] * ti0 + Qc[4 + i] * ti1;
      if (act) {
        st_cell256(psi + 4 * cell, p);
        if (r + 1 < ny)
          st_async_v2(out_line + 16u * static_cast<unsigned>(col), ty0 * p[0] + ty1 * p[2], ty0 * p[1] + ty1 * p[3],
                      out_bar + 8u * k);
      }
    }
  }
  cluster_barrier();  // (every hand-off was consumed; the CTAs leave together)
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

void launch_sweep_prefactor(const SweepArgs& a, double* table, long long stride, cudaStream_t s, int planes) {
  if (a.n <= 0) return;
  if (planes != kPrefDoubles && planes != kPrefMinvDoubles) throw std::invalid_argument("sweep_prefactor: planes");
  const long long ncell = static_cast<long long>(a.nx) * a.ny;
  sweep_prefactor_kernel<<<dim3(static_cast<unsigned>((ncell + 255) / 256), a.n), 256, 0, s>>>(a, table, stride,
                                                                                               planes);
  RTLR_CUDA(cudaGetLastError());
}

namespace {

constexpr size_t kScanSmemMax = 220 * 1024;  // dynamic shared memory per block (<= 227 KB with the static part)

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encode_tiled() {
  static const EncodeTiled fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeTiled>(p);
  }();
  return fn;
}

// The sources of all n directions as a 2-D tensor of 128-byte rows (16
// doubles = 4 cells); a chunk is a 16 x 32 box (128 cells), 128-byte swizzle.
bool make_source_map(const SweepArgs& a, CUtensorMap* m) {
  const EncodeTiled enc = encode_tiled();
  if (!enc) return false;
  const unsigned long long total = static_cast<unsigned long long>(a.n - 1) * a.rhs_stride +
                                   4ull * static_cast<unsigned long long>(a.nx) * a.ny;
  const cuuint64_t dims[2] = {16, (total + 15) / 16};
  const cuuint64_t strides[1] = {128};
  const cuuint32_t box[2] = {16, static_cast<cuuint32_t>(kWChunk / 4)};
  const cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(a.rhs), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// psi of all n directions as the same kind of tensor (for the TMA store).
bool make_psi_map(const SweepArgs& a, CUtensorMap* m) {
  const EncodeTiled enc = encode_tiled();
  if (!enc || a.psi_stride % 16 != 0 || reinterpret_cast<uintptr_t>(a.psi) % 16 != 0) return false;
  const unsigned long long total = static_cast<unsigned long long>(a.n - 1) * a.psi_stride +
                                   4ull * static_cast<unsigned long long>(a.nx) * a.ny;
  if (total % 16 != 0) return false;  // (a box past the last row would be clipped: keep whole rows)
  const cuuint64_t dims[2] = {16, total / 16};
  const cuuint64_t strides[1] = {128};
  const cuuint32_t box[2] = {16, static_cast<cuuint32_t>(kWChunk / 4)};
  const cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, a.psi, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

}  // namespace

void launch_sweep_scan(const SweepArgs& a_in, bool uniform, cudaStream_t s) {
  SweepArgs a = a_in;
  // RTLR_SCAN_STOUT: 0 the lanes store their own cells, 1 read-back and
  // coalesced stores, 2 TMA stores of whole chunks (A/B)
  static const int stage_out = [] {
    const char* e = std::getenv("RTLR_SCAN_STOUT");
    return e ? std::max(0, std::min(2, std::atoi(e))) : 2;
  }();
  a.stage_out = stage_out;
  if (a.n <= 0) return;
  // Launch plan for a chunk width (64 cells, or 128 for the wide kernel).
  struct Plan {
    int mode = kOne, W = 1, nck = 1, linew = 0;
    bool smem_lines = true;
    size_t smem = 0;  // groups' dynamic shared memory
  };
  auto plan_for = [&](bool wide) {
    const int ch = wide ? kWChunk : kChunk;
    const int nchunk = (a.nx + ch - 1) / ch;
    auto lines_fit = [&](int linew) {
      return static_cast<size_t>(kWarps) * 2 * line_pitch_w(linew, wide) * sizeof(double) <= kLineSmemBudget;
    };
    // Last-wave fill of n*c warps over the resident warp slots (SMs x blocks/SM x kWarps).
    auto wave_eff = [&](int c, int linew, bool smem_lines) {
      const size_t smem = static_cast<size_t>(kWarps / c) * group_doubles(c, linew, smem_lines, wide) * sizeof(double);
      const int per_sm = std::max(1, std::min(uniform ? 1 : 2, static_cast<int>((227u * 1024u) / (smem + 1024u))));
      const double slots = static_cast<double>(sm_count()) * per_sm * kWarps;
      const double waves = static_cast<double>(a.n) * c / slots;
      return waves <= 1.0 ? waves : waves / std::ceil(waves);
    };
    // Warps per direction W in {1, 2, 4, 8}, best last-wave fill, ties keep
    // the smaller W.  Rows whose full-width trace lines fit shared memory
    // (nx <= 768): row interleave (at most one warp per 2 rows).  Wider
    // rows: column segments (every segment non-empty, lines of one segment
    // in shared memory); only if no split fits do the lines go to L2.
    Plan p;
    p.nck = nchunk;
    p.linew = a.nx;
    p.smem_lines = lines_fit(a.nx);
    double best = -1.0;
    if (p.smem_lines) {
      // (c <= nchunk: the row chain of ny + nchunk - 1 dependent steps stays
      // shorter than a warp's own ny / c rows x nchunk steps)
      for (int c = 1; c <= kWarps && (c == 1 || (2 * c <= a.ny && c <= nchunk)); c *= 2) {
        const double eff = wave_eff(c, a.nx, true);
        if (eff > best + 1e-3) best = eff, p.W = c;
      }
      p.mode = p.W > 1 ? kRows : kOne;
    } else {
      for (int c = 2; c <= kWarps; c *= 2) {
        const int k = (nchunk + c - 1) / c;
        if ((c - 1) * k >= nchunk || !lines_fit(k * ch)) continue;
        const double eff = wave_eff(c, k * ch, true);
        if (eff > best + 1e-3) best = eff, p.W = c, p.nck = k;
      }
      if (p.W > 1) {
        p.mode = kSplit;
        p.smem_lines = true;
        p.linew = p.nck * ch;
      } else {  // rows in L2
        for (int c = 1; c <= kWarps && (c == 1 || 2 * c <= a.ny); c *= 2) {
          const double eff = wave_eff(c, a.nx, false);
          if (eff > best + 1e-3) best = eff, p.W = c;
        }
        p.mode = p.W > 1 ? kRows : kOne;
      }
    }
    static const int forced_w = [] {  // RTLR_SCAN_W: warps per direction for row-interleaved plans (tuning)
      const char* e = std::getenv("RTLR_SCAN_W");
      const int v = e ? std::atoi(e) : 0;
      return (v == 1 || v == 2 || v == 4 || v == 8) ? v : 0;
    }();
    if (forced_w && p.mode != kSplit && (forced_w == 1 || 2 * forced_w <= a.ny)) {
      p.W = forced_w;
      p.mode = forced_w > 1 ? kRows : kOne;
    }
    p.smem = static_cast<size_t>(kWarps / p.W) * group_doubles(p.W, p.linew, p.smem_lines, wide) * sizeof(double);
    return p;
  };
  // Uniform media take the wide kernel when the rows of the source tensor
  // (128 B = 4 cells) line up with the chunks, rows are at least one chunk
  // wide, the trace lines sit in shared memory and a ring of >= 2 tiles fits.
  CUtensorMap tmap;
  std::memset(&tmap, 0, sizeof(tmap));
  const char* te = std::getenv("RTLR_SWEEP_TMA");
  bool wide = uniform && !(te && te[0] == '0') && a.nx >= kWChunk && a.nx % 4 == 0 && a.rhs_stride % 16 == 0 &&
              reinterpret_cast<uintptr_t>(a.rhs) % 16 == 0;
  Plan pl;
  int stages = 0;
  if (wide) {
    pl = plan_for(true);
    const size_t room = kScanSmemMax > pl.smem + 1024 ? kScanSmemMax - pl.smem - 1024 : 0;
    static const int max_stages = [] {  // RTLR_SCAN_STAGES: cap on the TMA ring depth (tuning)
      const char* e = std::getenv("RTLR_SCAN_STAGES");
      const int v = e ? std::atoi(e) : 0;
      return v >= 2 && v <= kMaxStages ? v : kMaxStages;
    }();
    stages = static_cast<int>(std::min<size_t>(max_stages, room / (static_cast<size_t>(kWarps) * kWTileBytes)));
    // Wide steps are longer: only when the directions (nearly) fill the
    // resident warp slots, i.e. the sweep is bandwidth-bound; a latency-bound
    // sweep of a few directions keeps the 64-cell steps (C5 256^2 x 256:
    // 0.25 ms narrow vs 0.46 ms wide; 512^2 x 1024, 86% of the slots: 3.22 ms
    // wide vs 3.28 ms narrow).  RTLR_SWEEP_TMA=1 forces the wide kernel
    // wherever it applies, =0 disables it.
    const bool fills = (te && te[0] == '1') ||
                       4LL * a.n * pl.W >= 3LL * sm_count() * kWarps;
    wide = fills && pl.smem_lines && stages >= 2 && make_source_map(a, &tmap);
  }
  CUtensorMap pmap;
  std::memset(&pmap, 0, sizeof(pmap));
  if (wide && a.stage_out == 2 && !(stages >= 3 && make_psi_map(a, &pmap))) a.stage_out = 1;
  size_t smem;
  if (wide) {
    smem = pl.smem + 1024 + static_cast<size_t>(kWarps) * stages * kWTileBytes;
  } else {
    pl = plan_for(false);
    smem = pl.smem;
  }
  const int W = pl.W, mode = pl.mode, nck = pl.nck;
  const bool smem_lines = pl.smem_lines;
  const int groups = kWarps / W;
  const int blocks = (a.n + groups - 1) / groups;
  auto go = [&](auto kern) {
    RTLR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kScanSmemMax)));
    kern<<<blocks, kWarps * 32, smem, s>>>(a, W, smem_lines, nck, stages, tmap, pmap);
  };
  const bool bc = a.bc != nullptr;
#define RTLR_SCAN_GO(U, M)                                                                        \
  (wide ? (bc ? go(sweep_scan_kernel<U, M, true, U>) : go(sweep_scan_kernel<U, M, false, U>))   \
        : (bc ? go(sweep_scan_kernel<U, M, true, false>) : go(sweep_scan_kernel<U, M, false, false>)))
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


namespace {

size_t wave_smem(int nx) {
  const int nchunk = (nx + 31) / 32;
  return (kConsts + static_cast<size_t>(kWaveWarps) * nchunk + static_cast<size_t>(kWaveWarps) * 2 * nx) *
         sizeof(double);
}

template <class F>
void wave_dispatch(bool uniform, bool bc, F&& go) {
  if (uniform)
    bc ? go(sweep_wave_kernel<true, true>) : go(sweep_wave_kernel<true, false>);
  else
    bc ? go(sweep_wave_kernel<false, true>) : go(sweep_wave_kernel<false, false>);
}

template <class K>
cudaLaunchConfig_t wave_config(K kern, int cluster, int nclusters, size_t smem, cudaStream_t s,
                               cudaLaunchAttribute* at) {
  RTLR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  if (cluster > 8) RTLR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(nclusters) * cluster);
  cfg.blockDim = dim3(kWaveWarps * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cluster;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cfg;
}

}  // namespace

int sweep_wave_cluster(const SweepArgs& a, bool uniform) {
  if (a.n <= 0 || wave_smem(a.nx) > kWaveSmemMax) return 0;
  // Largest cluster (8, 4, 2 CTAs) of which all n fit on the GPU at once
  // (the query accounts for GPC placement); cached per kernel and row width.
  static std::vector<std::pair<long long, int>> cache;  // key -> max active clusters
  const bool bc = a.bc != nullptr;
  for (int cs = 8; cs >= 2; cs /= 2) {
    const long long key = ((static_cast<long long>(a.nx) * 4 + (uniform ? 2 : 0) + (bc ? 1 : 0)) << 5) | cs;
    int fit = -1;
    for (auto& e : cache)
      if (e.first == key) fit = e.second;
    if (fit < 0) {
      wave_dispatch(uniform, bc, [&](auto kern) {
        cudaLaunchAttribute at[1];
        const cudaLaunchConfig_t cfg = wave_config(kern, cs, 1, wave_smem(a.nx), nullptr, at);
        RTLR_CUDA(cudaOccupancyMaxActiveClusters(&fit, kern, &cfg));
      });
      cache.push_back({key, fit});
    }
    if (fit >= a.n) return cs;
  }
  return 0;
}

void launch_sweep_wave(const SweepArgs& a, bool uniform, int cluster, cudaStream_t s) {
  if (a.n <= 0) return;
  if (!uniform && a.pref == nullptr) throw std::logic_error("sweep_wave: general media need the M^-1 table");
  if (cluster == 0) cluster = sweep_wave_cluster(a, uniform);
  if (cluster < 1 || cluster > 16) throw std::invalid_argument("sweep_wave: cluster size must be 1..16");
  const size_t smem = wave_smem(a.nx);
  if (smem > kWaveSmemMax) throw std::invalid_argument("sweep_wave: rows too wide for the shared-memory trace lines");
  wave_dispatch(uniform, a.bc != nullptr, [&](auto kern) {
    cudaLaunchAttribute at[1];
    const cudaLaunchConfig_t cfg = wave_config(kern, cluster, a.n, smem, s, at);
    RTLR_CUDA(cudaLaunchKernelEx(&cfg, kern, a, cluster));
  });
  RTLR_CUDA(cudaGetLastError());
}

}  // namespace cuda
}  // namespace rtlr
