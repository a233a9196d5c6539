// K3 — streaming-operator stencil: StreamingOperator::apply
// (proj/src/operators.cpp:283-288) and the fused residual-norm epilogue used
// by the greedy selection and the all-angle verification
// (proj/src/low_rank.cpp:202-215, 283-307).
//
// Per DOF row the sum runs over the stored CSR entries in column order
// (upwind neighbour block before or after the diagonal block, exact zeros
// skipped) without FMA contraction, so apply() is bitwise the reference's.
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

// grid = (kResidParts, m): block (p, k) sums squares of the residual of
// angle k over the rows p, p + P*256, ... in a fixed pattern.
__global__ void residual_partials(const StencilArgs A, const int* __restrict__ angles,
                                  const double* __restrict__ dirs, const double* __restrict__ Y,
                                  long long ldy, const double* __restrict__ rhs,
                                  const double* __restrict__ bc, long long bc_stride,
                                  double* __restrict__ work) {
  __shared__ double sh[32];
  const int k = blockIdx.y;
  const int ang = angles ? angles[k] : k;
  const double omx = dirs[3 * ang], omy = dirs[3 * ang + 1];
  const double* y = Y + k * ldy;
  const double* g = bc ? bc + ang * bc_stride : nullptr;
  const int ndof = 4 * A.ncell;
  double acc = 0.0;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < ndof; r += gridDim.x * blockDim.x) {
    const int c = r >> 2;
    double res = rhs[r] - apply_row(A, c % A.nx, c / A.nx, r & 3, omx, omy, y);
    if (g) res += g[r];
    acc += res * res;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double s = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) work[static_cast<size_t>(k) * gridDim.x + blockIdx.x] = s;
  }
}

__global__ void residual_finish(int m, int parts, const double* __restrict__ work,
                                double* __restrict__ norms) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  double s = 0.0;
  for (int p = 0; p < parts; ++p) s += work[static_cast<size_t>(k) * parts + p];
  norms[k] = sqrt(s);
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
  for (int k0 = 0; k0 < m; k0 += 65535) {
    const int mk = (m - k0 < 65535) ? m - k0 : 65535;
    residual_partials<<<dim3(kResidParts, mk), 256, 0, s>>>(
        a, d_angles ? d_angles + k0 : nullptr, d_dirs, Y + k0 * ldy, ldy, rhs, bc, bc_stride,
        work + static_cast<size_t>(k0) * kResidParts);
    RTLR_CUDA(cudaGetLastError());
  }
  residual_finish<<<(m + 127) / 128, 128, 0, s>>>(m, kResidParts, work, norms);
  RTLR_CUDA(cudaGetLastError());
}

}  // namespace cuda
}  // namespace rtlr
