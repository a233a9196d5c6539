// K1 for heterogeneous media and many directions (replaces rtlr::sweep,
// proj/src/sweep.cpp:9-57, batched): the full-rank SI-DSA sweeps of C3/C4
// and any large heterogeneous batch.
//
// Why a separate kernel.  In a heterogeneous medium every (cell, direction)
// needs its own 4x4 solve with the cell's Sigma_t block (128 B).  Reading
// that block once per update from L2, one lane per mesh row, made the
// skewed wavefront (sweep.cu) L1TEX-bound at ~10% of HBM.  Here
//   * one warp sweeps D directions of the same quadrant at once (lane i owns
//     row i of a 32-row band, skewed diagonal wavefront as in sweep.cu), so
//     each Sigma_t block and source cell a lane loads serves D updates;
//   * Sigma_t and the (shared) source are read from a skewed copy of the
//     mesh (per quadrant orientation, built once per problem / per call):
//     at a step the 32 lanes' cells are contiguous, so every 16-byte plane
//     of them is one coalesced 512-byte cp.async burst into a shared-memory
//     queue instead of 32 scattered sectors;
//   * the cell block M = Omega_x Ax + Omega_y Ay + Sigma_t has a positive
//     definite symmetric part (Ax + Ax^T = t_R t_R^T + t_L t_L^T >= 0, Sigma_t
//     a sigma-weighted mass matrix; operators.cpp:47-79), so Gaussian
//     elimination needs no pivoting (stable, pivots > 0): ~90 fp64 operations
//     per update with fp64 reciprocals (MUFU seed + two Newton steps);
//   * the scalar flux can be accumulated in the epilogue (sum_j w_j psi_j over
//     the warp's directions, one partial per direction group, reduced in a
//     fixed order afterwards), so the full-rank iteration never writes psi.
// Results agree with the reference's pivoted LU to rounding (the parity
// tests hold them to 1e-12 per direction).  The singular-block error
// (sweep.cpp:49-52) is raised for a non-positive pivot or a non-finite
// solution: for the positive-real blocks of a valid problem the pivots are
// bounded below by the smallest eigenvalue of the symmetric part, so the
// reference's relative test min|U_ii| <= 1e-14 max|M| cannot fire there.
#include <algorithm>
#include <cstring>
#include <stdexcept>
#include <type_traits>

#include "device.cuh"
#include "sweep_het.cuh"

namespace rtlr {
namespace cuda {

namespace {

constexpr int kQ = 4;        // queue depth (steps in flight per warp)
constexpr int kPlanes = 10;  // 16-byte planes per lane per step: Sigma_t (8) + source (2)
// queue slot bytes: the planes of 32 lanes, then lane 0's prefetched
// y-inflow traces of the step (kHetD x 16 bytes)
constexpr int kSlotBytes = kPlanes * 512 + kHetD * 16;
constexpr int kPublish = 2;  // columns per published progress update

__device__ __forceinline__ double rcp64(double x) {
  // MUFU seed (~2^-23) + two Newton steps: correctly rounded to ~1 ulp
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}

__device__ __forceinline__ void cp16(unsigned dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ double2 lds2(unsigned a) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ void st_cell256(double* p, double a, double b, double c, double d) {
  asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}
__device__ __forceinline__ void ld_cell(const double* p, double v[4]) {
  asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
               : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
               : "l"(p));
}

// Per-direction constants in shared memory (broadcast reads):
// d0..d3 (diagonal of Omega_x Ax + Omega_y Ay), cx10, cx01, cy10, cy01
// (its off-diagonal entries), kx0, kx1, ky0, ky1 (upwind couplings), w.
constexpr int kDirConsts = 14;  // (13 used, even for 16-byte loads)

// Natural cell of lane position (band b, diagonal d, lane i) for orientation (xu, yu); -1 if padding.
__host__ __device__ __forceinline__ long long skew_cell(int nx, int ny, bool xu, bool yu, int b, int d, int i) {
  const int r = b * 32 + i, c = d - i;
  if (r >= ny || c < 0 || c >= nx) return -1;
  const int rn = yu ? r : ny - 1 - r, cn = xu ? c : nx - 1 - c;
  return static_cast<long long>(rn) * nx + cn;
}

// dst[o][b][d][p][i] (16-byte planes) from src cells of `planes` 16-byte
// planes (AoS, cell-major), zero where the position is padding.
__global__ void skew_layout_kernel(int nx, int ny, int nb, int dp, int planes, const double2* __restrict__ src,
                                   double2* __restrict__ dst, int o_begin, int o_end) {
  const long long per_o = static_cast<long long>(nb) * dp * planes * 32;
  const long long total = per_o * (o_end - o_begin);
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(e & 31);
    long long q = e >> 5;
    const int p = static_cast<int>(q % planes);
    q /= planes;
    const int d = static_cast<int>(q % dp);
    q /= dp;
    const int b = static_cast<int>(q % nb);
    const int o = o_begin + static_cast<int>(q / nb);
    const long long cell = skew_cell(nx, ny, (o & 1) == 0, (o & 2) == 0, b, d, i);
    dst[e] = cell < 0 ? make_double2(0.0, 0.0) : src[cell * planes + p];
  }
}

// phi[dof] = sum over groups (fixed order) of part[g][dof]
__global__ void reduce_parts_kernel(long long ndof, int groups, const double* __restrict__ part, double* __restrict__ phi) {
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < ndof;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    double s = 0.0;
    for (int g = 0; g < groups; ++g) s += part[static_cast<long long>(g) * ndof + e];
    phi[e] = s;
  }
}

template <int D, bool MULTI, bool HAS_BC, bool WPSI, bool WPHI>
__global__ void __launch_bounds__(256, 1) sweep_het_kernel(const SweepHetArgs a) {
  extern __shared__ __align__(16) double smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int W = a.W;
  const int groups = 8 / W;
  const int gl = wib / W, w = wib % W;
  const int grp = blockIdx.x * groups + gl;
  if (grp >= a.ngroups) return;  // a whole group exits together
  const int nx = a.nx, ny = a.ny, nb = (ny + 31) >> 5, S = nx > 32 ? nx : 32, dp = S + 31;
  // shared memory: per-warp queues, then per-group constants and counters
  double* queue = smem + static_cast<size_t>(wib) * kQ * (kSlotBytes / 8);  // slot s, plane p: 32 lanes x 2 doubles
  double* gbase = smem + static_cast<size_t>(8) * kQ * (kSlotBytes / 8) + static_cast<size_t>(gl) * (D * kDirConsts + 8);
  double* dc = gbase;                                             // D x kDirConsts
  volatile int* prod = reinterpret_cast<volatile int*>(gbase + D * kDirConsts);  // W counters
  const int orient = a.group_orient[grp];
  const bool xu = (orient & 1) == 0, yu = (orient & 2) == 0;
  // orientation constants: outflow traces and the 2x2 streaming blocks
  const double* tx = xu ? a.sc.trx_r : a.sc.trx_l;
  const double* ty = yu ? a.sc.try_r : a.sc.try_l;
  const double tx0 = tx[0], tx1 = tx[1], ty0 = ty[0], ty1 = ty[1];
  if (w == 0) {
    if (lane < D) {
      const int slot = grp * D + lane;
      const int ang = a.slot_angle[slot];
      double* c = dc + lane * kDirConsts;
      if (ang < 0) {
        for (int k = 0; k < kDirConsts; ++k) c[k] = 0.0;
        c[0] = c[1] = c[2] = c[3] = 1.0;  // identity block for padding slots (results unused)
        int* ci = reinterpret_cast<int*>(c + 13);
        ci[0] = -1;
        ci[1] = 0;
      } else {
        const double omx = a.dirs[3 * ang], omy = a.dirs[3 * ang + 1];
        const double* ax = xu ? a.sc.ax_minus : a.sc.ax_plus;  // 4x4 tensorized, column-major
        const double* ay = yu ? a.sc.ay_minus : a.sc.ay_plus;
        // (Omega_x Ax + Omega_y Ay) entries, operators.cpp:61-79 tensorization
        c[0] = omx * ax[0] + omy * ay[0];
        c[1] = omx * ax[5] + omy * ay[5];
        c[2] = omx * ax[10] + omy * ay[10];
        c[3] = omx * ax[15] + omy * ay[15];
        c[4] = omx * ax[1];   // (1,0)
        c[5] = omx * ax[4];   // (0,1)
        c[6] = omy * ay[2];   // (2,0)
        c[7] = omy * ay[8];   // (0,2)
        c[8] = omx * (xu ? -a.sc.trx_l[0] : a.sc.trx_r[0]);
        c[9] = omx * (xu ? -a.sc.trx_l[1] : a.sc.trx_r[1]);
        c[10] = omy * (yu ? -a.sc.try_l[0] : a.sc.try_r[0]);
        c[11] = omy * (yu ? -a.sc.try_l[1] : a.sc.try_r[1]);
        c[12] = a.slot_weight ? a.slot_weight[slot] : 0.0;
        int* ci = reinterpret_cast<int*>(c + 13);
        ci[0] = a.slot_pos[slot];
        ci[1] = ang;
      }
    }
    if (lane < W) prod[lane] = 0;
  }
  asm volatile("bar.sync %0, %1;" ::"r"(gl + 1), "r"(W * 32) : "memory");
  // the skewed Sigma_t / source copies of this orientation
  const double2* sig = reinterpret_cast<const double2*>(a.sig_skew) + static_cast<long long>(orient) * nb * dp * 8 * 32;
  const double2* src = reinterpret_cast<const double2*>(a.rhs_skew) + static_cast<long long>(orient) * nb * dp * 2 * 32;
  double* lines = a.line + static_cast<long long>(grp) * W * D * nx * 2;
  double* my_line = lines + static_cast<long long>(w) * D * nx * 2;
  const int pw = (w + W - 1) % W;
  const double* in_line = lines + static_cast<long long>(pw) * D * nx * 2;
  double* part = WPHI ? a.phi_part + static_cast<long long>(grp) * a.ndof : nullptr;
  const int kw = (w < nb) ? (nb - w + W - 1) / W : 0;  // bands of this warp
  const int total = kw * S + 31;
  const unsigned qbase = static_cast<unsigned>(__cvta_generic_to_shared(queue)) + lane * 16;

  // lane stream: k-th band of the warp, column col (skew: col = t - lane - k S).
  // Lane 0 also prefetches the step's y-inflow traces (the band below, from
  // the producer warp's line) when they are already published; otherwise it
  // waits for them at the step itself.
  int seen = 0;  // MULTI: producer progress already observed
  int f0k = 0, f0c = 0;  // lane 0's prefetch position (band ordinal, column), warp-uniform
  const bool own_pf = !MULTI && S > 31 + kQ;  // W = 1: own line, written >= S - 31 steps earlier
  unsigned pfm = 0;  // bit s: slot s holds lane 0's prefetched traces
  auto fill = [&](int slot, int k, int col) {
    const unsigned q = qbase + slot * kSlotBytes;
    const bool ok = k < kw && col >= 0 && col < S;
    const int band = w + k * W;
    const long long pos = ok ? (static_cast<long long>(band) * dp + (col + lane)) : 0;
    const double2* s8 = sig + pos * 8 * 32 + lane;
    const double2* s2 = src + pos * 2 * 32 + lane;
#pragma unroll
    for (int p = 0; p < 8; ++p) cp16(q + p * 512, s8 + p * 32);
    cp16(q + 8 * 512, s2);
    cp16(q + 9 * 512, s2 + 32);
    // Lane 0's traces for that step: the band below, column f0c of the
    // producer's line.  The position (f0k, f0c) is lane 0's, kept in every
    // lane, so the wait below is taken by the whole warp together (a lane-0
    // spin would leave the warp diverged for the solves that follow).  The
    // wait happens here, kQ steps ahead: the consumer trails its producer by
    // the lane skew plus the queue depth and the traces arrive by cp.async,
    // off the step's critical path.
    pfm &= ~(1u << slot);
    if (f0k < kw && f0c < nx && w + f0k * W > 0) {
      if (MULTI) {
        const int gidx = (w > 0 ? f0k : f0k - 1) * nx + f0c;  // ordinal of band - 1 in warp pw
        if (seen <= gidx) {
          while ((seen = prod[pw]) <= gidx) {
          }
        }
        __threadfence_block();
      }
      if (MULTI || own_pf) {
        if (lane == 0) {
          const unsigned ql = qbase + slot * kSlotBytes + kPlanes * 512;
#pragma unroll
          for (int d = 0; d < D; ++d) cp16(ql + d * 16, in_line + (static_cast<long long>(d) * nx + f0c) * 2);
        }
        pfm |= 1u << slot;
      }
    }
    if (++f0c == S) {
      f0c = 0;
      ++f0k;
    }
  };
  int pk = 0, pcol = -lane;  // prefetch stream position
#pragma unroll
  for (int s = 0; s < kQ; ++s) {
    fill(s, pk, pcol);
    cp_commit();
    if (++pcol == S) {
      pcol = 0;
      ++pk;
    }
  }
  int ck = 0, ccol = -lane;  // compute stream position
  double txi[D][2], tyo[D][2];
#pragma unroll
  for (int k = 0; k < D; ++k) txi[k][0] = txi[k][1] = tyo[k][0] = tyo[k][1] = 0.0;
  for (int t0 = 0; t0 < total; t0 += kQ) {
#pragma unroll 1
    for (int s = 0; s < kQ; ++s) {
      if (t0 + s >= total) break;  // warp-uniform
      cp_wait<kQ - 1>();
      const unsigned q = qbase + s * kSlotBytes;
      double m[16];
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        const double2 v = lds2(q + p * 512);
        m[2 * p] = v.x;
        m[2 * p + 1] = v.y;
      }
      const double2 r01 = lds2(q + 8 * 512), r23 = lds2(q + 9 * 512);
      // y inflow traces: from lane - 1's previous step
      double yi[D][2];
#pragma unroll
      for (int k = 0; k < D; ++k) {
        yi[k][0] = __shfl_up_sync(0xffffffffu, tyo[k][0], 1);
        yi[k][1] = __shfl_up_sync(0xffffffffu, tyo[k][1], 1);
      }
      const int band = w + ck * W;
      const int row = band * 32 + lane;
      const bool act = ck < kw && ccol >= 0 && ccol < nx && row < ny;
      const int col = ccol;
      if (lane == 0 && act) {  // lane 0: the band below's traces
        if (band == 0) {
#pragma unroll
          for (int k = 0; k < D; ++k) yi[k][0] = yi[k][1] = 0.0;
        } else if (pfm & (1u << s)) {
#pragma unroll
          for (int k = 0; k < D; ++k) {
            const double2 v = lds2(q + kPlanes * 512 + k * 16);
            yi[k][0] = v.x;
            yi[k][1] = v.y;
          }
        } else {
          if (MULTI) {
            const int gidx = (w > 0 ? ck : ck - 1) * nx + col;
            if (seen <= gidx) {
              while ((seen = prod[pw]) <= gidx) {
              }
              __threadfence_block();
            }
          }
#pragma unroll
          for (int k = 0; k < D; ++k) {
            const double2 v = __ldcg(reinterpret_cast<const double2*>(in_line + (static_cast<long long>(k) * nx + col) * 2));
            yi[k][0] = v.x;
            yi[k][1] = v.y;
          }
        }
      }
      fill(s, pk, pcol);
      cp_commit();
      if (++pcol == S) {
        pcol = 0;
        ++pk;
      }
      // reconverge before the cell solves (lane 0 may have waited for its
      // producer above; diverged lanes would run the solves twice)
      __syncwarp();
      if (act) {
        if (col == 0) {
#pragma unroll
          for (int k = 0; k < D; ++k) txi[k][0] = txi[k][1] = 0.0;
        }
        const int rn = yu ? row : ny - 1 - row, cn = xu ? col : nx - 1 - col;
        const long long cell = static_cast<long long>(rn) * nx + cn;
        double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
        int sgn = 0;
#pragma unroll
        for (int k = 0; k < D; ++k) {
          const double* c = dc + k * kDirConsts;
          const double2 c01 = *reinterpret_cast<const double2*>(c), c23 = *reinterpret_cast<const double2*>(c + 2);
          const double2 c45 = *reinterpret_cast<const double2*>(c + 4), c67 = *reinterpret_cast<const double2*>(c + 6);
          const double2 c89 = *reinterpret_cast<const double2*>(c + 8), cab = *reinterpret_cast<const double2*>(c + 10);
          double wk = c[12];
          double v0 = r01.x, v1 = r01.y, v2 = r23.x, v3 = r23.y;
          const int* ci = reinterpret_cast<const int*>(c + 13);
          if (HAS_BC) {
            double g[4];
            ld_cell(a.bc + static_cast<long long>(ci[1]) * a.bc_stride + 4 * cell, g);
            v0 += g[0];
            v1 += g[1];
            v2 += g[2];
            v3 += g[3];
          }
          // local = rhs - Omega_x Bx psi_x - Omega_y By psi_y   (sweep.cpp:40-46)
          v0 -= c89.x * txi[k][0];
          v1 -= c89.y * txi[k][0];
          v2 -= c89.x * txi[k][1];
          v3 -= c89.y * txi[k][1];
          v0 -= cab.x * yi[k][0];
          v1 -= cab.x * yi[k][1];
          v2 -= cab.y * yi[k][0];
          v3 -= cab.y * yi[k][1];
          // M = Omega_x Ax + Omega_y Ay + Sigma_t (column-major a_ij = A[j*4+i])
          double a00 = m[0] + c01.x, a10 = m[1] + c45.x, a20 = m[2] + c67.x, a30 = m[3];
          double a01 = m[4] + c45.y, a11 = m[5] + c01.y, a21 = m[6], a31 = m[7] + c67.x;
          double a02 = m[8] + c67.y, a12 = m[9], a22 = m[10] + c23.x, a32 = m[11] + c45.x;
          double a03 = m[12], a13 = m[13] + c67.y, a23 = m[14] + c45.y, a33 = m[15] + c23.y;
          // elimination without pivoting
          const double r0 = rcp64(a00);
          const double l1 = a10 * r0, l2 = a20 * r0, l3 = a30 * r0;
          a11 -= l1 * a01;
          a21 -= l2 * a01;
          a31 -= l3 * a01;
          a12 -= l1 * a02;
          a22 -= l2 * a02;
          a32 -= l3 * a02;
          a13 -= l1 * a03;
          a23 -= l2 * a03;
          a33 -= l3 * a03;
          v1 -= l1 * v0;
          v2 -= l2 * v0;
          v3 -= l3 * v0;
          const double r1 = rcp64(a11);
          const double m2 = a21 * r1, m3 = a31 * r1;
          a22 -= m2 * a12;
          a32 -= m3 * a12;
          a23 -= m2 * a13;
          a33 -= m3 * a13;
          v2 -= m2 * v1;
          v3 -= m3 * v1;
          const double r2 = rcp64(a22);
          const double n3 = a32 * r2;
          a33 -= n3 * a23;
          v3 -= n3 * v2;
          const double r3 = rcp64(a33);
          const double p3 = v3 * r3;
          const double p2 = (v2 - a23 * p3) * r2;
          const double p1 = (v1 - a12 * p2 - a13 * p3) * r1;
          const double p0 = (v0 - a01 * p1 - a02 * p2 - a03 * p3) * r0;
          // pivots of a positive-real block are positive: the sign bits of the
          // four pivots (integer pipe); a zero or tiny pivot shows as a
          // non-finite solution, caught once per step below
          sgn |= __double2hiint(a00) | __double2hiint(a11) | __double2hiint(a22) | __double2hiint(a33);
          if (WPSI) {
            const int pos = ci[0];
            if (pos >= 0) st_cell256(a.psi + static_cast<long long>(pos) * a.psi_stride + 4 * cell, p0, p1, p2, p3);
          }
          if (!WPHI) wk = 1.0;  // (psi-only launch: acc carries the finiteness test)
          acc0 += wk * p0;
          acc1 += wk * p1;
          acc2 += wk * p2;
          acc3 += wk * p3;
          // outflow traces: x (per y-mode) for the next cell of the row,
          // y (per x-mode) for the row above
          txi[k][0] = tx0 * p0 + tx1 * p1;
          txi[k][1] = tx0 * p2 + tx1 * p3;
          tyo[k][0] = ty0 * p0 + ty1 * p2;
          tyo[k][1] = ty0 * p1 + ty1 * p3;
        }
        // singular-block test (sweep.cpp:49-52): a non-positive pivot, or a
        // non-finite solution (acc sums w_k psi_k; with zero weights 0 * inf is NaN)
        if (sgn < 0 || !isfinite(acc0 + acc1 + acc2 + acc3)) atomicExch(a.err, 1);
        if (WPHI) st_cell256(part + 4 * cell, acc0, acc1, acc2, acc3);
        if (lane == 31 && band + 1 < nb) {
#pragma unroll
          for (int k = 0; k < D; ++k)
            __stcg(reinterpret_cast<double2*>(my_line + (static_cast<long long>(k) * nx + col) * 2),
                   make_double2(tyo[k][0], tyo[k][1]));
          if (MULTI && ((col + 1) % kPublish == 0 || col + 1 == nx)) {
            __threadfence_block();
            prod[w] = ((band - w) / W) * nx + col + 1;
          }
        }
      } else {
#pragma unroll
        for (int k = 0; k < D; ++k) tyo[k][0] = tyo[k][1] = 0.0;
      }
      __syncwarp();
      if (++ccol == S) {
        ccol = 0;
        ++ck;
      }
    }
  }
  cp_wait<0>();
}

// the handoff between a group's warps is deadlock free when a row is longer
// than the lane skew of the warp chain (as in sweep.cu)
bool multi_ok(int W, int S) { return 32 * W + 2 * kPublish < S; }

}  // namespace

void build_skew_layout(int nx, int ny, const double* cells, int planes, double* out, cudaStream_t s) {
  const int nb = (ny + 31) / 32, S = nx > 32 ? nx : 32, dp = S + 31;
  const long long total = 4LL * nb * dp * planes * 32;
  const int grid = static_cast<int>(std::min<long long>((total + 255) / 256, 148LL * 32));
  skew_layout_kernel<<<grid, 256, 0, s>>>(nx, ny, nb, dp, planes, reinterpret_cast<const double2*>(cells),
                                          reinterpret_cast<double2*>(out), 0, 4);
  RTLR_CUDA(cudaGetLastError());
}

size_t skew_layout_doubles(int nx, int ny, int planes) {
  const int nb = (ny + 31) / 32, S = nx > 32 ? nx : 32;
  return static_cast<size_t>(4) * nb * (S + 31) * planes * 32 * 2;
}

int sweep_het_warps(int nx, int ny, int ngroups) {
  const int nb = (ny + 31) / 32, S = nx > 32 ? nx : 32;
  // warps per group: fill ~148 x 8 warp slots, at most one per band, within the deadlock bound
  int W = 1;
  while (W < 8 && static_cast<long long>(ngroups) * W * 2 <= 148 * 8 && 2 * W <= nb && multi_ok(2 * W, S)) W *= 2;
  return W;
}

void launch_sweep_het(const SweepHetArgs& a, cudaStream_t s) {
  if (a.ngroups <= 0) return;
  const int groups_per_block = 8 / a.W;
  const int blocks = (a.ngroups + groups_per_block - 1) / groups_per_block;
  const size_t smem = (static_cast<size_t>(8) * kQ * (kSlotBytes / 8) +
                       static_cast<size_t>(groups_per_block) * (kHetD * kDirConsts + 8)) *
                      sizeof(double);
  auto go = [&](auto kern) {
    RTLR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    kern<<<blocks, 256, smem, s>>>(a);
  };
  // instantiations: the full-rank iteration (scalar flux, no psi), psi only
  // (the converged sweep, rtlr_cu_sweep), both; with and without inflow
  const bool bc = a.bc != nullptr, psi = a.psi != nullptr, phi = a.phi_part != nullptr;
  if (!psi && !phi) throw std::invalid_argument("sweep_het: neither psi nor phi requested");
  const int mode = (psi ? 1 : 0) + (phi ? 2 : 0);
  auto pick = [&](auto multi) {
    constexpr bool M = decltype(multi)::value;
    if (bc) {
      if (mode == 1) go(sweep_het_kernel<kHetD, M, true, true, false>);
      else if (mode == 2) go(sweep_het_kernel<kHetD, M, true, false, true>);
      else go(sweep_het_kernel<kHetD, M, true, true, true>);
    } else {
      if (mode == 1) go(sweep_het_kernel<kHetD, M, false, true, false>);
      else if (mode == 2) go(sweep_het_kernel<kHetD, M, false, false, true>);
      else go(sweep_het_kernel<kHetD, M, false, true, true>);
    }
  };
  if (a.W > 1)
    pick(std::true_type{});
  else
    pick(std::false_type{});
  RTLR_CUDA(cudaGetLastError());
}

void reduce_phi_parts(long long ndof, int groups, const double* part, double* phi, cudaStream_t s) {
  const int grid = static_cast<int>(std::min<long long>((ndof + 255) / 256, 148LL * 16));
  reduce_parts_kernel<<<grid, 256, 0, s>>>(ndof, groups, part, phi);
  RTLR_CUDA(cudaGetLastError());
}

}  // namespace cuda
}  // namespace rtlr
