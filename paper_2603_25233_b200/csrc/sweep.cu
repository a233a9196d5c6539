// K1 — batched transport sweep (replaces rtlr::sweep, proj/src/sweep.cpp:9-57).
//
// One warp per direction.  Lane i owns mesh rows i, i+32, i+64, ... (in the
// direction's upwind order) and runs a skewed diagonal wavefront: at step t
// lane i processes virtual position v = t - i, i.e. band v / S, column
// v % S with S = max(nx, 32).  Because the upwind couplings of the K = 1
// upwind DG operator are rank one per axis (b^- = -t_L t_R^T,
// operators.cpp:47-57), a cell only needs the two outflow-trace
// coefficients of each upwind neighbour:
//   * x-upwind traces stay in the lane's registers (previous cell of its row);
//   * y-upwind traces come from lane i-1 one step earlier (__shfl_up_sync);
//   * lane 0 reads the traces lane 31 wrote for the band below from a small
//     per-direction line buffer (L2-resident, S-31 steps later).
// Each lane step moves one 32-byte cell of rhs in and one of psi out.
//
// Cell arithmetic follows the reference: local = rhs - Omega_x*Bx*psi_x -
// Omega_y*By*psi_y, block = Omega_x*Ax + Omega_y*Ay + Sigma_t,c, partial-pivot
// LU (first maximum), singular test min|U_ii| <= 1e-14 max|block| -> error.
// When every Sigma_t block is bitwise identical (homogeneous medium, C5)
// the block is the same for all cells of a direction: it is factored once
// per warp into an explicit inverse and each cell is a 4x4 mat-vec.
#include "device.cuh"

namespace rtlr {
namespace cuda {

namespace {

__device__ __forceinline__ void ld_cell(const double* p, double v[4]) {
  const double2* q = reinterpret_cast<const double2*>(p);
  const double2 a = __ldg(q), b = __ldg(q + 1);
  v[0] = a.x;
  v[1] = a.y;
  v[2] = b.x;
  v[3] = b.y;
}

// Streaming source read: each lane walks its mesh row 32 B per step, so ask
// L2 to fetch 256 B per miss (the lane's next 8 cells) instead of one 32-B
// sector; consecutive steps then hit L2 and DRAM sees full bursts.
__device__ __forceinline__ void ld_cell_stream(const double* p, double v[4]) {
  asm volatile("ld.global.nc.L2::256B.v2.f64 {%0, %1}, [%4];\n\t"
               "ld.global.nc.L2::256B.v2.f64 {%2, %3}, [%4+16];"
               : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
               : "l"(p));
}

__device__ __forceinline__ void st_cell(double* p, const double v[4]) {
  double2* q = reinterpret_cast<double2*>(p);
  __stcs(q, make_double2(v[0], v[1]));
  __stcs(q + 1, make_double2(v[2], v[3]));
}

#define A_(i, j) A[(j) * 4 + (i)]

// Swap rows k and p of the 4x4 column-major A and of b using predicated
// selects only (indices are compile-time constants after unrolling).
template <int K>
__device__ __forceinline__ void pivot_rows(double* A, double* b, int p) {
#pragma unroll
  for (int i = K + 1; i < 4; ++i) {
    const bool s = (p == i);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const double x = A_(K, j), y = A_(i, j);
      A_(K, j) = s ? y : x;
      A_(i, j) = s ? x : y;
    }
    const double x = b[K], y = b[i];
    b[K] = s ? y : x;
    b[i] = s ? x : y;
  }
}

template <int K>
__device__ __forceinline__ int argmax_col(const double* A) {
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
__device__ __forceinline__ void eliminate(double* A, double* b) {
  const double inv = 1.0 / A_(K, K);
#pragma unroll
  for (int i = K + 1; i < 4; ++i) {
    const double l = A_(i, K) * inv;
#pragma unroll
    for (int j = K + 1; j < 4; ++j) A_(i, j) -= l * A_(K, j);
    b[i] -= l * b[K];
  }
}

// Solves A x = b in place (b <- x).  Returns false on a singular block
// under the reference's test (sweep.cpp:49-52).
__device__ __forceinline__ bool lu_solve4(double* A, double* b) {
  double amax = 0.0;
#pragma unroll
  for (int k = 0; k < 16; ++k) amax = fmax(amax, fabs(A[k]));
  int p;
  p = argmax_col<0>(A);
  pivot_rows<0>(A, b, p);
  eliminate<0>(A, b);
  p = argmax_col<1>(A);
  pivot_rows<1>(A, b, p);
  eliminate<1>(A, b);
  p = argmax_col<2>(A);
  pivot_rows<2>(A, b, p);
  eliminate<2>(A, b);
  const double dmin = fmin(fmin(fabs(A_(0, 0)), fabs(A_(1, 1))), fmin(fabs(A_(2, 2)), fabs(A_(3, 3))));
  // back substitution (column oriented, as Eigen's triangular solve)
#pragma unroll
  for (int i = 3; i >= 0; --i) {
    b[i] = b[i] / A_(i, i);
#pragma unroll
    for (int j = 0; j < i; ++j) b[j] -= b[i] * A_(j, i);
  }
  return dmin > 1e-14 * amax;
}

// Explicit inverse of a 4x4 via the same pivoted LU applied to e_0..e_3.
__device__ __forceinline__ bool invert4(const double* M, double* Minv) {
  bool ok = true;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    double A[16], e[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int k = 0; k < 16; ++k) A[k] = M[k];
    e[c] = 1.0;
    ok = lu_solve4(A, e) && ok;
#pragma unroll
    for (int r = 0; r < 4; ++r) Minv[c * 4 + r] = e[r];
  }
  return ok;
}

#undef A_

// rhs cells in flight per lane (smem queue): deeper for the single-warp
// throughput kernel, shallower when trace lines share the smem budget.
template <bool MULTI>
__host__ __device__ constexpr int prefetch_depth() { return MULTI ? 4 : 8; }
constexpr int kQueueSlotDoubles = 32 * 4 + 2;  // 32 lanes x one cell + the lane-0 trace pair

// Source cells stream through a per-warp shared-memory queue filled with
// cp.async: in-flight data costs no registers and the wait is explicit.
// dst: this lane's slot entry; the two 16-byte halves of the cell go 512
// bytes apart so a warp's LDS.128 / smem fill is contiguous (no conflicts)
__device__ __forceinline__ void cp_cell_async(double* dst_smem, const double* src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst_smem));
  asm volatile(
      "cp.async.cg.shared.global.L2::256B [%0], [%1], 16;\n\t"
      "cp.async.cg.shared.global.L2::256B [%2], [%3], 16;" ::"r"(d),
      "l"(src), "r"(d + 512), "l"(src + 2)
      : "memory");
}
__device__ __forceinline__ void cp16_async(double* dst_smem, const double* src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst_smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void st_cell256(double* p, const double v[4]) {
  // one 32-byte cell per lane per instruction (STG.E.ENL2.256): lanes walk
  // different rows, so L1TEX wavefronts per warp store halve vs 2 x 128-bit
  asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(v[0]), "d"(v[1]), "d"(v[2]),
               "d"(v[3])
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
constexpr int kLineSmemBudget = 64 * 1024;  // bytes of trace lines per block kept in smem
constexpr int kPublish = 2;                 // columns per published progress update

// Shared-memory load the compiler may not hoist out of the step loop (keeps
// the per-direction 4x4 inverse out of the register file).
__device__ __forceinline__ double2 lds2(const double* p) {
  double2 v;
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(p));
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
  return v;
}

__device__ __forceinline__ void lds_cell(const double* p, double v[4]) {
  const double2 a = lds2(p), b = lds2(p + 64);
  v[0] = a.x;
  v[1] = a.y;
  v[2] = b.x;
  v[3] = b.y;
}

// Shared memory of one direction group (W warps).  Warp w hands the top
// traces of each of its bands to warp (w+1) % W through a full-row trace
// line (nx x 2 doubles, in smem when it fits, else in L2) plus a progress
// counter: slot col of line w is only rewritten (band b+W) after warp w+1
// read it for band b+1, because that rewrite depends on the read through
// the upwind chain band b+1 -> ... -> b+W.  Readers therefore only wait for
// data to be published; there are no space waits and no cycles.  With a
// single warp per direction the line is the warp's own and needs no counter.
struct GroupSmem {
  double* consts;      // 40: minv / dstream (16), kx ky tx ty (8), spare
  volatile int* prod;  // W: columns published by warp w's lane 31
  double* lines;       // W x nx x 2 (shared or global)
};

__host__ __device__ constexpr int group_smem_doubles(int W, int nx, bool smem_lines) {
  // even, so every group's constants stay 16-byte aligned for ld.shared.v2
  return 40 + 2 * ((W + 3) / 4) + (smem_lines ? W * nx * 2 : 0);
}

// A lane's position in its warp's stream of work: the k-th band owned by
// the warp (band = w + k W) and a column (negative during the initial lane
// skew, >= nx in the padding up to S).  cell is linear in col, so it is
// advanced incrementally and only recomputed at band changes.
struct Stream {
  long long cell;
  int col, k, band;
  bool rowok;
};

struct Walk {
  int nx, ny, nb, S, w, W, lane, xs;
  bool xu, yu;
  __device__ __forceinline__ void seek(Stream& s, int k, int col) const {
    s.k = k;
    s.col = col;
    s.band = w + k * W;
    const int row = s.band * 32 + lane;
    s.rowok = s.band < nb && row < ny;
    const int cb = yu ? row : ny - 1 - row;
    const int ca = xu ? col : nx - 1 - col;
    s.cell = static_cast<long long>(cb) * nx + ca;
  }
  __device__ __forceinline__ void step(Stream& s) const {
    ++s.col;
    s.cell += xs;
    if (s.col == S) seek(s, s.k + 1, 0);
  }
  __device__ __forceinline__ bool active(const Stream& s) const {
    return s.rowok && s.col >= 0 && s.col < nx;
  }
};

template <bool UNIFORM, bool MULTI, bool HAS_BC>
__global__ void __launch_bounds__(256, 2) sweep_kernel(const SweepArgs a, int W, bool smem_lines) {
  constexpr int kPrefetch = prefetch_depth<MULTI>();
  extern __shared__ double smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int groups = (blockDim.x >> 5) / W;
  const int g = wib / W, w = wib % W;
  const int slot = blockIdx.x * groups + g;
  if (slot >= a.n || g >= groups) return;  // a whole direction group exits together
  // per-warp source queue: kPrefetch slots x (32 lanes x 4 doubles + 2)
  double* wqueue = smem + static_cast<size_t>(wib) * kPrefetch * kQueueSlotDoubles;
  double* queue = wqueue + static_cast<size_t>(lane) * 2;  // halves at +0 and +64 doubles
  GroupSmem sm;
  {
    double* base = smem + static_cast<size_t>(blockDim.x >> 5) * kPrefetch * kQueueSlotDoubles +
                   static_cast<size_t>(g) * group_smem_doubles(W, a.nx, smem_lines);
    sm.consts = base;
    sm.prod = reinterpret_cast<int*>(base + 40);
    sm.lines = smem_lines ? base + 40 + 2 * ((W + 3) / 4) : a.line + static_cast<size_t>(slot) * W * a.nx * 2;
  }
  const int ang = a.angles ? a.angles[slot] : slot;
  const double omx = a.dirs[3 * ang], omy = a.dirs[3 * ang + 1];
  const bool xu = omx >= 0.0, yu = omy >= 0.0;  // sweep.cpp:37-38
  // Per-direction constants, computed once by warp 0 into shared memory:
  // the cell block Omega_x Ax + Omega_y Ay (general path) or the inverse of
  // Omega_x Ax + Omega_y Ay + Sigma_t (uniform medium), and the upwind
  // couplings (B psi_up)[my,mx] = c[mx] * (t . psi_up[my,:]) with
  // (c, t) = (-t_L, t_R) for the "minus" blocks and (t_R, t_L) for "plus".
  if (w == 0) {
    const double* ax = xu ? a.sc.ax_minus : a.sc.ax_plus;
    const double* ay = yu ? a.sc.ay_minus : a.sc.ay_plus;
    if (lane < 16) {
      const double d = omx * ax[lane] + omy * ay[lane];
      sm.consts[lane] = UNIFORM ? d + a.sigma_t[lane] : d;
    }
    if (lane < 2) {
      sm.consts[16 + lane] = omx * (xu ? -a.sc.trx_l[lane] : a.sc.trx_r[lane]);
      sm.consts[18 + lane] = xu ? a.sc.trx_r[lane] : a.sc.trx_l[lane];
      sm.consts[20 + lane] = omy * (yu ? -a.sc.try_l[lane] : a.sc.try_r[lane]);
      sm.consts[22 + lane] = yu ? a.sc.try_r[lane] : a.sc.try_l[lane];
    }
    __syncwarp();
    if (UNIFORM && lane == 0) {
      double M[16], Mi[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) M[k] = sm.consts[k];
      if (!invert4(M, Mi)) atomicExch(a.err, 1);
#pragma unroll
      for (int k = 0; k < 16; ++k) sm.consts[k] = Mi[k];
    }
    if (lane < W) sm.prod[lane] = 0;
  }
  // all W warps of the group see the constants and initialised counters
  asm volatile("bar.sync %0, %1;" ::"r"(g + 1), "r"(W * 32) : "memory");
  const double* cst = sm.consts;
  const double kx[2] = {cst[16], cst[17]}, tx[2] = {cst[18], cst[19]};
  const double ky[2] = {cst[20], cst[21]}, ty[2] = {cst[22], cst[23]};

  Walk walk;
  walk.nx = a.nx;
  walk.ny = a.ny;
  walk.nb = (a.ny + 31) >> 5;
  walk.S = a.nx > 32 ? a.nx : 32;
  walk.w = w;
  walk.W = W;
  walk.lane = lane;
  walk.xu = xu;
  walk.yu = yu;
  walk.xs = xu ? 1 : -1;
  const int S = walk.S, nx = a.nx, nb = walk.nb;
  const int kw = (w < nb) ? (nb - w + W - 1) / W : 0;  // bands of this warp
  const int total = kw * S + 31;
  const double* rhs = a.rhs + static_cast<long long>(slot) * a.rhs_stride;
  const double* bc = HAS_BC ? a.bc + static_cast<long long>(ang) * a.bc_stride : nullptr;
  double* psi = a.psi + static_cast<long long>(slot) * a.psi_stride;
  const int pw = (w + W - 1) % W;  // producer of our lane 0's traces
  double* my_line = sm.lines + static_cast<size_t>(w) * nx * 2;
  const double* in_line = sm.lines + static_cast<size_t>(pw) * nx * 2;
  // single warp: lane 0's traces (written by its own lane 31, S-31 steps
  // earlier) ride in the same cp.async group as the source cell
  const bool line_pf = !MULTI && (S - 31 > kPrefetch);

  // prefetch queue: rhs of steps t .. t+kPrefetch-1 (slot = step % kPrefetch).
  // Idle positions load a valid dummy cell (never consumed).
  Stream cur, pre;
  walk.seek(cur, 0, -lane);
  walk.seek(pre, 0, -lane);
#pragma unroll
  for (int s = 0; s < kPrefetch; ++s) {
    cp_cell_async(queue + s * kQueueSlotDoubles, rhs + (walk.active(pre) ? 4 * pre.cell : 0));
    if (line_pf && lane == 0 && walk.active(pre) && pre.band > 0)
      cp16_async(wqueue + s * kQueueSlotDoubles + 128, in_line + 2 * pre.col);
    cp_commit();
    walk.step(pre);
  }

  double txi0 = 0.0, txi1 = 0.0;  // x traces of the previous cell in the row
  double tyo0 = 0.0, tyo1 = 0.0;  // y traces produced last step
  int seen = 0;                   // MULTI: producer progress already observed by lane 0
  for (int t0 = 0; t0 < total; t0 += kPrefetch) {
#pragma unroll
    for (int s = 0; s < kPrefetch; ++s) {
      if (t0 + s >= total) break;  // warp-uniform
      // the oldest of kPrefetch groups (this step's cell) has landed
      cp_wait<kPrefetch - 1>();
      double v[4];
      lds_cell(queue + s * kQueueSlotDoubles, v);
      double2 lq = make_double2(0.0, 0.0);
      if (line_pf && lane == 0) lq = lds2(wqueue + s * kQueueSlotDoubles + 128);
      __syncwarp();
      // refill this queue slot with the step kPrefetch ahead
      cp_cell_async(queue + s * kQueueSlotDoubles, rhs + (walk.active(pre) ? 4 * pre.cell : 0));
      if (line_pf && lane == 0 && walk.active(pre) && pre.band > 0)
        cp16_async(wqueue + s * kQueueSlotDoubles + 128, in_line + 2 * pre.col);
      cp_commit();
      walk.step(pre);
      double yi0 = __shfl_up_sync(0xffffffffu, tyo0, 1);
      double yi1 = __shfl_up_sync(0xffffffffu, tyo1, 1);
      tyo0 = 0.0;
      tyo1 = 0.0;
      const bool act = walk.active(cur);
      const int col = cur.col;
      if (act) {
        if (lane == 0) {
          if (cur.band == 0) {
            yi0 = yi1 = 0.0;
          } else {
            // traces of band-1, column col, from the producer warp's line
            if (MULTI) {
              const int gidx = ((cur.band - 1 - pw) / W) * nx + col;
              if (seen <= gidx) {
                while ((seen = sm.prod[pw]) <= gidx) {
                }
                __threadfence_block();
              }
            }
            const double* r = in_line + 2 * col;
            if (line_pf) {
              yi0 = lq.x;
              yi1 = lq.y;
            } else if (smem_lines) {
              yi0 = r[0];
              yi1 = r[1];
            } else {
              yi0 = __ldcg(r);
              yi1 = __ldcg(r + 1);
            }
          }
        }
        if (col == 0) {
          txi0 = 0.0;
          txi1 = 0.0;
        }
        if (HAS_BC) {
          double gb[4];
          ld_cell(bc + 4 * cur.cell, gb);
#pragma unroll
          for (int k = 0; k < 4; ++k) v[k] += gb[k];
        }
        // local = rhs - Omega_x Bx psi_x - Omega_y By psi_y   (sweep.cpp:40-46)
        v[0] = v[0] - kx[0] * txi0;
        v[1] = v[1] - kx[1] * txi0;
        v[2] = v[2] - kx[0] * txi1;
        v[3] = v[3] - kx[1] * txi1;
        v[0] = v[0] - ky[0] * yi0;
        v[1] = v[1] - ky[0] * yi1;
        v[2] = v[2] - ky[1] * yi0;
        v[3] = v[3] - ky[1] * yi1;
        double p[4];
        if (UNIFORM) {
          p[0] = p[1] = p[2] = p[3] = 0.0;
#pragma unroll
          for (int j = 0; j < 4; ++j) {  // column j of the inverse
            const double2 lo = lds2(cst + 4 * j), hi = lds2(cst + 4 * j + 2);
            p[0] += lo.x * v[j];
            p[1] += lo.y * v[j];
            p[2] += hi.x * v[j];
            p[3] += hi.y * v[j];
          }
        } else {
          double A[16];
          const double2* sb = reinterpret_cast<const double2*>(a.sigma_t + 16 * cur.cell);
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const double2 s2 = __ldg(sb + k);
            A[2 * k] = cst[2 * k] + s2.x;
            A[2 * k + 1] = cst[2 * k + 1] + s2.y;
          }
          if (!lu_solve4(A, v)) atomicExch(a.err, 1);
#pragma unroll
          for (int r = 0; r < 4; ++r) p[r] = v[r];
        }
        st_cell256(psi + 4 * cur.cell, p);
        // outflow traces: x (per y-mode) for the next cell of this row,
        // y (per x-mode) for the row above (next lane / next band).
        txi0 = tx[0] * p[0] + tx[1] * p[1];
        txi1 = tx[0] * p[2] + tx[1] * p[3];
        tyo0 = ty[0] * p[0] + ty[1] * p[2];
        tyo1 = ty[0] * p[1] + ty[1] * p[3];
        if (lane == 31 && cur.band + 1 < nb) {
          double* r = my_line + 2 * col;
          if (smem_lines) {
            r[0] = tyo0;
            r[1] = tyo1;
          } else {
            __stcg(r, tyo0);
            __stcg(r + 1, tyo1);
          }
          if (MULTI && ((col + 1) % kPublish == 0 || col + 1 == nx)) {
            __threadfence_block();
            sm.prod[w] = ((cur.band - w) / W) * nx + col + 1;
          }
        }
      }
      __syncwarp();
      walk.step(cur);
    }
  }
  cp_wait<0>();
}

// Handoff is deadlock free only when a band row is longer than the lane
// skew of the warp chain: warp j at step t needs warp j-1 past step t+32
// (plus the publish granularity), and warp 0's next band needs warp W-1.
__host__ __device__ constexpr bool multi_ok(int W, int S) { return 32 * W + 2 * kPublish < S; }

}  // namespace

void launch_sweep(const SweepArgs& a, bool uniform, cudaStream_t s) {
  if (a.n <= 0) return;
  // Warps per direction: enough concurrent warps to fill 148 SMs x 16, at
  // most one per 32-row band, at most 8, and within the deadlock bound.
  const int nb = (a.ny + 31) / 32;
  const int S = a.nx > 32 ? a.nx : 32;
  int W = 1;
  while (W < 8 && static_cast<long long>(a.n) * W * 2 <= 148 * 16 && 2 * W <= nb && multi_ok(2 * W, S)) W *= 2;
  const int warps_per_block = 8;
  const int groups = warps_per_block / W;
  const int blocks = (a.n + groups - 1) / groups;
  // W == 1 keeps its trace line in L2 (prefetched through the queue);
  // multi-warp groups share lines in smem when they fit.
  const bool smem_lines = W > 1 && static_cast<size_t>(8) * a.nx * 2 * sizeof(double) <= kLineSmemBudget;
  const int pf = W > 1 ? prefetch_depth<true>() : prefetch_depth<false>();
  const size_t smem = (static_cast<size_t>(warps_per_block) * pf * kQueueSlotDoubles +
                       static_cast<size_t>(groups) * group_smem_doubles(W, a.nx, smem_lines)) *
                      sizeof(double);
  auto go = [&](auto kern) {
    RTLR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    kern<<<blocks, warps_per_block * 32, smem, s>>>(a, W, smem_lines);
  };
  const bool bc = a.bc != nullptr;
  if (uniform) {
    if (W > 1)
      bc ? go(sweep_kernel<true, true, true>) : go(sweep_kernel<true, true, false>);
    else
      bc ? go(sweep_kernel<true, false, true>) : go(sweep_kernel<true, false, false>);
  } else {
    if (W > 1)
      bc ? go(sweep_kernel<false, true, true>) : go(sweep_kernel<false, true, false>);
    else
      bc ? go(sweep_kernel<false, false, true>) : go(sweep_kernel<false, false, false>);
  }
  RTLR_CUDA(cudaGetLastError());
}

namespace {

__device__ __forceinline__ double c5u(std::uint64_t seed, std::uint64_t counter) {
  std::uint64_t z = counter * 0x9E3779B97F4A7C15ull + seed;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return static_cast<double>(z >> 11) * 0x1.0p-53;
}

__global__ void c5_fill_kernel(double* rhs, long long total, long long base, std::uint64_t seed) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    rhs[i] = c5u(seed, static_cast<std::uint64_t>(base + i));
}

}  // namespace

void launch_c5_fill(double* rhs, long long n_dirs, long long dir0, long long ndof, std::uint64_t seed,
                    cudaStream_t s) {
  const long long total = n_dirs * ndof;
  if (total <= 0) return;
  c5_fill_kernel<<<148 * 8, 256, 0, s>>>(rhs, total, dir0 * ndof, seed);
  RTLR_CUDA(cudaGetLastError());
}

}  // namespace cuda
}  // namespace rtlr
