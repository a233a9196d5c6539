// K3 — streaming-operator stencil: StreamingOperator::apply
// (proj/src/operators.cpp:283-288) and the fused residual-norm epilogue used
// by the greedy selection and the all-angle verification
// (proj/src/low_rank.cpp:202-215, 283-307).
//
// Per DOF row the sum runs over the stored CSR entries in column order
// (upwind neighbour block before or after the diagonal block, exact zeros
// skipped) without FMA contraction, so apply() is bitwise the reference's.
#include <algorithm>

#include "device.cuh"

namespace rtlr {
namespace cuda {

namespace {

__device__ __forceinline__ double blk_row(const double* B, int i, const double* v, double tmp) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const double b = B[j * 4 + i];
    if (b != 0.0) tmp = __dadd_rn(tmp, __dmul_rn(b, v[j]));
  }
  return tmp;
}

// (Sigma_t + omx D_x + omy D_y) v, row i of cell (a, b).
__device__ __forceinline__ double apply_row(const StencilArgs& A, int a, int b, int i, double omx,
                                            double omy, const double* v) {
  const int c = b * A.nx + a;
  const double* vc = v + 4 * static_cast<size_t>(c);
  double out = blk_row(A.sigma_t + 16 * static_cast<size_t>(c), i, vc, 0.0);
  if (omx != 0.0) {
    double t = 0.0;
    if (omx >= 0.0) {  // D_x^-: west neighbour columns precede the diagonal
      if (a > 0) t = blk_row(A.sc.bx_minus, i, vc - 4, t);
      t = blk_row(A.sc.ax_minus, i, vc, t);
    } else {  // D_x^+: diagonal, then east neighbour
      t = blk_row(A.sc.ax_plus, i, vc, t);
      if (a + 1 < A.nx) t = blk_row(A.sc.bx_plus, i, vc + 4, t);
    }
    out = __dadd_rn(out, __dmul_rn(omx, t));
  }
  if (omy != 0.0) {
    double t = 0.0;
    const size_t up = 4 * static_cast<size_t>(A.nx);
    if (omy >= 0.0) {
      if (b > 0) t = blk_row(A.sc.by_minus, i, vc - up, t);
      t = blk_row(A.sc.ay_minus, i, vc, t);
    } else {
      t = blk_row(A.sc.ay_plus, i, vc, t);
      if (b + 1 < A.ny) t = blk_row(A.sc.by_plus, i, vc + up, t);
    }
    out = __dadd_rn(out, __dmul_rn(omy, t));
  }
  return out;
}

__global__ void stream_apply_kernel(const StencilArgs A, double omx, double omy,
                                    const double* __restrict__ v, double* __restrict__ out) {
  const int ndof = 4 * A.ncell;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < ndof; r += gridDim.x * blockDim.x) {
    const int c = r >> 2;
    out[r] = apply_row(A, c % A.nx, c / A.nx, r & 3, omx, omy, v);
  }
}

// Residual norms, one thread per cell and a group of RG angles per block row
// (blockIdx.y): the cell's Sigma_t block and source are loaded once (two
// 256-bit loads each... 16 + 4 doubles) and reused for the group's angles;
// each angle's expanded solution y_k is read as 32-byte cells (the upwind
// neighbours mostly from L1).  Row arithmetic is apply_row's (Sigma_t row,
// then the streaming terms in the CSR column order, no FMA contraction).
// Block (p, g) writes one partial per angle of the group; the per-angle sum
// over partials runs in a fixed order, independent of the angle's position
// in the batch, so equal columns give bitwise equal norms.
constexpr int kResidGroup = 4;
constexpr int kResidThreads = 256;

__device__ __forceinline__ void ld4(const double* p, double v[4]) {
  asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
               : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
               : "l"(p));
}

// out[i] (+)= sum_j B[j*4+i] v[j] over the nonzeros of a streaming block
__device__ __forceinline__ void blk_add(const double* B, const double v[4], double t[4]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) t[i] = blk_row(B, i, v, t[i]);
}

__global__ void __launch_bounds__(kResidThreads) residual_cells(const StencilArgs A, int m, const int* __restrict__ angles,
                                                                const double* __restrict__ dirs, const double* __restrict__ Y,
                                                                long long ldy, const double* __restrict__ rhs,
                                                                const double* __restrict__ bc, long long bc_stride,
                                                                double* __restrict__ work) {
  __shared__ double sh[kResidGroup][kResidThreads / 32];
  const int c = blockIdx.x * kResidThreads + threadIdx.x;
  const int k0 = blockIdx.y * kResidGroup;
  double acc[kResidGroup];
#pragma unroll
  for (int j = 0; j < kResidGroup; ++j) acc[j] = 0.0;
  if (c < A.ncell) {
    const int a = c % A.nx, b = c / A.nx;
    double S[16], r[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) ld4(A.sigma_t + 16 * static_cast<size_t>(c) + 4 * q, S + 4 * q);
    ld4(rhs + 4 * static_cast<size_t>(c), r);
    const size_t up = 4 * static_cast<size_t>(A.nx);
#pragma unroll
    for (int j = 0; j < kResidGroup; ++j) {
      const int k = k0 + j;
      if (k >= m) break;
      const int ang = angles ? angles[k] : k;
      const double omx = dirs[3 * ang], omy = dirs[3 * ang + 1];
      const double* y = Y + k * ldy + 4 * static_cast<size_t>(c);
      double v[4];
      ld4(y, v);
      double out[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) out[i] = blk_row(S, i, v, 0.0);
      if (omx != 0.0) {
        double t[4] = {0.0, 0.0, 0.0, 0.0}, w[4];
        if (omx >= 0.0) {  // D_x^-: west neighbour columns precede the diagonal
          if (a > 0) {
            ld4(y - 4, w);
            blk_add(A.sc.bx_minus, w, t);
          }
          blk_add(A.sc.ax_minus, v, t);
        } else {  // D_x^+: diagonal, then east neighbour
          blk_add(A.sc.ax_plus, v, t);
          if (a + 1 < A.nx) {
            ld4(y + 4, w);
            blk_add(A.sc.bx_plus, w, t);
          }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) out[i] = __dadd_rn(out[i], __dmul_rn(omx, t[i]));
      }
      if (omy != 0.0) {
        double t[4] = {0.0, 0.0, 0.0, 0.0}, w[4];
        if (omy >= 0.0) {
          if (b > 0) {
            ld4(y - up, w);
            blk_add(A.sc.by_minus, w, t);
          }
          blk_add(A.sc.ay_minus, v, t);
        } else {
          blk_add(A.sc.ay_plus, v, t);
          if (b + 1 < A.ny) {
            ld4(y + up, w);
            blk_add(A.sc.by_plus, w, t);
          }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) out[i] = __dadd_rn(out[i], __dmul_rn(omy, t[i]));
      }
      double g[4] = {0.0, 0.0, 0.0, 0.0};
      if (bc) ld4(bc + static_cast<long long>(ang) * bc_stride + 4 * static_cast<size_t>(c), g);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        double res = __dsub_rn(r[i], out[i]);
        if (bc) res = __dadd_rn(res, g[i]);
        acc[j] = __fma_rn(res, res, acc[j]);
      }
    }
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < kResidGroup; ++j) {
    double v = acc[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) sh[j][wid] = v;
  }
  __syncthreads();
  if (threadIdx.x < kResidGroup) {
    const int k = k0 + threadIdx.x;
    if (k < m) {
      double s = 0.0;
      for (int w = 0; w < kResidThreads / 32; ++w) s += sh[threadIdx.x][w];
      work[static_cast<size_t>(k) * gridDim.x + blockIdx.x] = s;
    }
  }
}

__global__ void residual_finish(int m, int parts, const double* __restrict__ work,
                                double* __restrict__ norms) {
  // one warp per angle: lanes stride the partials, fixed shuffle tree
  const int k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (k >= m) return;
  double s = 0.0;
  for (int p = lane; p < parts; p += 32) s += work[static_cast<size_t>(k) * parts + p];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) norms[k] = sqrt(s);
}

}  // namespace

void launch_stream_apply(const StencilArgs& a, double omx, double omy, const double* v, double* out,
                         cudaStream_t s) {
  const int ndof = 4 * a.ncell;
  int grid = (ndof + 255) / 256;
  if (grid > 148 * 16) grid = 148 * 16;
  stream_apply_kernel<<<grid, 256, 0, s>>>(a, omx, omy, v, out);
  RTLR_CUDA(cudaGetLastError());
}

void launch_residual_norms(const StencilArgs& a, int m, const int* d_angles, const double* d_dirs,
                           const double* Y, long long ldy, const double* rhs, const double* bc,
                           long long bc_stride, double* work, double* norms, cudaStream_t s) {
  if (m <= 0) return;
  const int parts = residual_parts(a.ncell);
  for (int k0 = 0; k0 < m; k0 += 65535 * kResidGroup) {
    const int mk = std::min(m - k0, 65535 * kResidGroup);
    residual_cells<<<dim3(parts, (mk + kResidGroup - 1) / kResidGroup), kResidThreads, 0, s>>>(
        a, mk, d_angles ? d_angles + k0 : nullptr, d_dirs, Y + k0 * ldy, ldy, rhs, bc, bc_stride,
        work + static_cast<size_t>(k0) * parts);
    RTLR_CUDA(cudaGetLastError());
  }
  residual_finish<<<(m * 32 + 255) / 256, 256, 0, s>>>(m, parts, work, norms);
  RTLR_CUDA(cudaGetLastError());
}

int residual_parts(int ncell) { return (ncell + kResidThreads - 1) / kResidThreads; }

}  // namespace cuda
}  // namespace rtlr
