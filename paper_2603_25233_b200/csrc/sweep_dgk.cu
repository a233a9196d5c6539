// Transport sweep and streaming operator for DG degree K != 1 (s = (K+1)^2
// DOFs per cell, K = 0 and 2..4): proj/src/sweep.cpp:10-57 and
// StreamingOperator::apply (proj/src/operators.cpp:283-288) for any K
// (proj/tests/test_sweep.cpp:142-155 sweeps quadratic elements).  The
// K = 1 hot path has its own kernels (sweep_scan.cu, sweep.cu,
// sweep_het.cu); this one is the general-degree path: one CTA per
// direction walks the cell anti-diagonals (every cell of a diagonal only
// needs the previous diagonal's outflow), one thread per cell forms the
// upwind right-hand side, the s x s block Omega_x A_x + Omega_y A_y +
// Sigma_t(cell), its partial-pivot LU (first maximum, the reference's
// singular test 1e-14 max|block|) and solve, in the reference's operation
// order.  The eight streaming blocks sit in shared memory.
#include <algorithm>
#include <stdexcept>
#include <string>

#include "sweep_dgk.cuh"

namespace rtlr {
namespace cuda {

namespace {

template <int S>
__global__ void __launch_bounds__(128) sweep_dgk_kernel(DgkSweepArgs a) {
  __shared__ double blk[8 * S * S];
  for (int e = threadIdx.x; e < 8 * S * S; e += blockDim.x) blk[e] = a.blocks[e];
  __syncthreads();
  const int k = blockIdx.x;
  const int ang = a.angles ? a.angles[k] : k;
  const double omx = a.dirs[3 * ang], omy = a.dirs[3 * ang + 1];
  const bool x_up = omx >= 0.0, y_up = omy >= 0.0;
  const double* ax = blk + (x_up ? 0 : 1) * S * S;
  const double* ay = blk + (y_up ? 2 : 3) * S * S;
  const double* bx = blk + (x_up ? 4 : 5) * S * S;
  const double* by = blk + (y_up ? 6 : 7) * S * S;
  const double* rhs = a.rhs + k * a.rhs_stride;
  const double* bc = a.bc ? a.bc + static_cast<long long>(ang) * a.bc_stride : nullptr;
  double* psi = a.psi + k * a.psi_stride;
  const int nx = a.nx, ny = a.ny;
  double lu[S * S], loc[S];
  int perm[S];
  for (int d = 0; d < nx + ny - 1; ++d) {
    const int ja0 = max(0, d - (ny - 1)), ja1 = min(d, nx - 1);
    for (int ja = ja0 + static_cast<int>(threadIdx.x); ja <= ja1; ja += blockDim.x) {
      const int jb = d - ja;
      const int ca = x_up ? ja : nx - 1 - ja, cb = y_up ? jb : ny - 1 - jb;
      const long long c = static_cast<long long>(cb) * nx + ca;
      for (int i = 0; i < S; ++i) loc[i] = bc ? rhs[c * S + i] + bc[c * S + i] : rhs[c * S + i];
      if (ja > 0) {  // upwind x neighbour, solved on the previous diagonal
        const double* up = psi + (c + (x_up ? -1 : 1)) * S;
        for (int i = 0; i < S; ++i) {
          double t = 0.0;
          for (int j = 0; j < S; ++j) t += bx[i + j * S] * up[j];
          loc[i] -= omx * t;
        }
      }
      if (jb > 0) {
        const double* up = psi + (c + (y_up ? -nx : nx)) * S;
        for (int i = 0; i < S; ++i) {
          double t = 0.0;
          for (int j = 0; j < S; ++j) t += by[i + j * S] * up[j];
          loc[i] -= omy * t;
        }
      }
      const double* st = a.sigma_t + c * S * S;
      double amax = 0.0;
      for (int e = 0; e < S * S; ++e) {
        lu[e] = omx * ax[e] + omy * ay[e] + st[e];
        amax = fmax(amax, fabs(lu[e]));
      }
      // partial-pivot LU, first maximum (Eigen PartialPivLU)
      for (int kk = 0; kk < S; ++kk) {
        int piv = kk;
        double big = fabs(lu[kk + kk * S]);
        for (int i = kk + 1; i < S; ++i)
          if (fabs(lu[i + kk * S]) > big) {
            big = fabs(lu[i + kk * S]);
            piv = i;
          }
        perm[kk] = piv;
        if (big != 0.0) {
          if (piv != kk)
            for (int j = 0; j < S; ++j) {
              const double t = lu[kk + j * S];
              lu[kk + j * S] = lu[piv + j * S];
              lu[piv + j * S] = t;
            }
          const double dd = lu[kk + kk * S];
          for (int i = kk + 1; i < S; ++i) lu[i + kk * S] /= dd;
        }
        for (int j = kk + 1; j < S; ++j) {
          const double u = lu[kk + j * S];
          for (int i = kk + 1; i < S; ++i) lu[i + j * S] -= lu[i + kk * S] * u;
        }
      }
      double dmin = fabs(lu[0]);
      for (int i = 1; i < S; ++i) dmin = fmin(dmin, fabs(lu[i + i * S]));
      if (!(dmin > 1e-14 * amax)) atomicExch(a.err, 1);
      for (int kk = 0; kk < S; ++kk) {
        const double t = loc[kk];
        loc[kk] = loc[perm[kk]];
        loc[perm[kk]] = t;
      }
      for (int i = 0; i < S; ++i) {
        const double xi = loc[i];
        for (int j = i + 1; j < S; ++j) loc[j] -= xi * lu[j + i * S];
      }
      for (int i = S - 1; i >= 0; --i) {
        loc[i] /= lu[i + i * S];
        const double xi = loc[i];
        for (int j = 0; j < i; ++j) loc[j] -= xi * lu[j + i * S];
      }
      for (int i = 0; i < S; ++i) psi[c * S + i] = loc[i];
    }
    __syncthreads();  // this diagonal's outflow is the next one's inflow
  }
}

// out = Sigma_t v + Omega_x (D_x v) + Omega_y (D_y v), one thread per cell
// row block; the sparse products sum in column order as the reference's CSR.
template <int S>
__global__ void apply_dgk_kernel(int nx, int ny, const double* __restrict__ sigma_t,
                                 const double* __restrict__ blocks, double omx, double omy,
                                 const double* __restrict__ v, double* __restrict__ out) {
  const long long ncell = static_cast<long long>(nx) * ny;
  const bool x_up = omx >= 0.0, y_up = omy >= 0.0;
  const double* ax = blocks + (x_up ? 0 : 1) * S * S;
  const double* ay = blocks + (y_up ? 2 : 3) * S * S;
  const double* bx = blocks + (x_up ? 4 : 5) * S * S;
  const double* by = blocks + (y_up ? 6 : 7) * S * S;
  for (long long c = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; c < ncell;
       c += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int ca = static_cast<int>(c % nx), cb = static_cast<int>(c / nx);
    const double* st = sigma_t + c * S * S;
    const bool has_xn = x_up ? ca > 0 : ca + 1 < nx;
    const bool has_yn = y_up ? cb > 0 : cb + 1 < ny;
    const double* vx = v + (c + (x_up ? -1 : 1)) * S;
    const double* vy = v + (c + (y_up ? -nx : nx)) * S;
    const double* vc = v + c * S;
    for (int i = 0; i < S; ++i) {
      double o = 0.0;
      for (int j = 0; j < S; ++j) o += st[i + j * S] * vc[j];
      if (omx != 0.0) {
        double t = 0.0;
        if (x_up) {  // D_x^-: west block (lower columns) first
          if (has_xn)
            for (int j = 0; j < S; ++j) t += bx[i + j * S] * vx[j];
          for (int j = 0; j < S; ++j) t += ax[i + j * S] * vc[j];
        } else {  // D_x^+: own block, then east
          for (int j = 0; j < S; ++j) t += ax[i + j * S] * vc[j];
          if (has_xn)
            for (int j = 0; j < S; ++j) t += bx[i + j * S] * vx[j];
        }
        o += omx * t;
      }
      if (omy != 0.0) {
        double t = 0.0;
        if (y_up) {
          if (has_yn)
            for (int j = 0; j < S; ++j) t += by[i + j * S] * vy[j];
          for (int j = 0; j < S; ++j) t += ay[i + j * S] * vc[j];
        } else {
          for (int j = 0; j < S; ++j) t += ay[i + j * S] * vc[j];
          if (has_yn)
            for (int j = 0; j < S; ++j) t += by[i + j * S] * vy[j];
        }
        o += omy * t;
      }
      out[c * S + i] = o;
    }
  }
}

template <int S>
void launch_sweep(const DgkSweepArgs& a, cudaStream_t s) {
  sweep_dgk_kernel<S><<<a.n, 128, 0, s>>>(a);
}

template <int S>
void launch_apply(int nx, int ny, const double* st, const double* blocks, double omx, double omy, const double* v,
                  double* out, cudaStream_t s) {
  const long long ncell = static_cast<long long>(nx) * ny;
  const int grid = static_cast<int>(std::min<long long>((ncell + 127) / 128, 148LL * 16));
  apply_dgk_kernel<S><<<grid, 128, 0, s>>>(nx, ny, st, blocks, omx, omy, v, out);
}

}  // namespace

void sweep_dgk(int degree, const DgkSweepArgs& a, cudaStream_t s) {
  if (a.n <= 0) return;
  switch (degree) {
    case 0: launch_sweep<1>(a, s); break;
    case 1: launch_sweep<4>(a, s); break;
    case 2: launch_sweep<9>(a, s); break;
    case 3: launch_sweep<16>(a, s); break;
    case 4: launch_sweep<25>(a, s); break;
    default: throw std::invalid_argument("sweep: DG degree " + std::to_string(degree) + " not built");
  }
  RTLR_CUDA(cudaGetLastError());
}

void apply_dgk(int degree, int nx, int ny, const double* sigma_t, const double* blocks, double omx, double omy,
               const double* v, double* out, cudaStream_t s) {
  switch (degree) {
    case 0: launch_apply<1>(nx, ny, sigma_t, blocks, omx, omy, v, out, s); break;
    case 1: launch_apply<4>(nx, ny, sigma_t, blocks, omx, omy, v, out, s); break;
    case 2: launch_apply<9>(nx, ny, sigma_t, blocks, omx, omy, v, out, s); break;
    case 3: launch_apply<16>(nx, ny, sigma_t, blocks, omx, omy, v, out, s); break;
    case 4: launch_apply<25>(nx, ny, sigma_t, blocks, omx, omy, v, out, s); break;
    default: throw std::invalid_argument("apply: DG degree " + std::to_string(degree) + " not built");
  }
  RTLR_CUDA(cudaGetLastError());
}

}  // namespace cuda
}  // namespace rtlr
