// Vector kernels of the SI-DSA outer loop (K2, K10, K13) and the DSA
// solve (K12): block-diagonal Sigma_s SpMV, scalar-flux accumulation,
// deterministic difference norms, BSR SpMV on the SIP-DG matrix and a
// block-Jacobi preconditioned CG.
//
// Every reduction is deterministic: a fixed grid writes one partial per
// block and consumers sum the partials in a fixed order, so reruns are
// bitwise identical (proj/tests/test_low_rank.cpp:441-470 contract).
#include <cstdlib>
#include "linalg.cuh"
#include "mg.cuh"

namespace rtlr {
namespace cuda {

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ double block_sum(double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x < 32) {
    s = (lane < (blockDim.x >> 5)) ? sh[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  }
  return s;  // valid in thread 0
}

__device__ __forceinline__ double block_max(double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x < 32) {
    s = (lane < (blockDim.x >> 5)) ? sh[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s = fmax(s, __shfl_xor_sync(0xffffffffu, s, o));
  }
  return s;
}

// Sum of n partials in a fixed order, computed identically by every block.
__device__ __forceinline__ double sum_partials(const double* part, int n, double* sh) {
  double v = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) v += part[i];
  v = block_sum(v, sh);
  if (threadIdx.x == 0) sh[32] = v;
  __syncthreads();
  const double r = sh[32];
  __syncthreads();
  return r;
}

// out = Sigma_s x (+ g): per DOF row, stored block entries in column order
// (Eigen row-major SpMV, operators.cpp:283 / full_rank.cpp:81), without FMA
// contraction so the result is bitwise the reference's.
__global__ void sigma_apply_kernel(int ndof, const double* __restrict__ blocks,
                                   const double* __restrict__ x, const double* __restrict__ x_minus,
                                   const double* __restrict__ g, double* __restrict__ out) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < ndof; r += gridDim.x * blockDim.x) {
    const int c = r >> 2, i = r & 3;
    const double* B = blocks + 16 * static_cast<size_t>(c);
    double tmp = 0.0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const double bij = B[j * 4 + i];
      double xj = x[4 * c + j];
      if (x_minus) xj = __dsub_rn(xj, x_minus[4 * c + j]);
      if (bij != 0.0) tmp = __dadd_rn(tmp, __dmul_rn(bij, xj));
    }
    out[r] = g ? __dadd_rn(tmp, g[r]) : tmp;
  }
}

// phi[i] = sum_u W[u] psi[u][i] in a fixed angle order.
__global__ void phi_accum_kernel(int ndof, int nu, const double* __restrict__ psi, long long ld,
                                 const double* __restrict__ w, double* __restrict__ phi) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ndof; i += gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int u = 0; u < nu; ++u) acc += psi[u * ld + i] * w[u];
    phi[i] = acc;
  }
}

// Block partials of ||a-b||_2^2 and ||a-b||_inf.
__global__ void diff_norm_partials(int n, const double* __restrict__ a, const double* __restrict__ b,
                                   double* __restrict__ part2, double* __restrict__ partinf) {
  __shared__ double sh[40];
  double s = 0.0, m = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double d = a[i] - (b ? b[i] : 0.0);
    s += d * d;
    m = fmax(m, fabs(d));
  }
  s = block_sum(s, sh);
  if (threadIdx.x == 0) part2[blockIdx.x] = s;
  m = block_max(m, sh);
  if (threadIdx.x == 0) partinf[blockIdx.x] = m;
}

__global__ void finish_norms(int nparts, const double* part2, const double* partinf, double* out) {
  __shared__ double sh[40];
  double s = 0.0, m = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) {
    s += part2[i];
    m = fmax(m, partinf[i]);
  }
  s = block_sum(s, sh);
  m = block_max(m, sh);
  if (threadIdx.x == 0) {
    out[0] = sqrt(s);
    out[1] = m;
  }
}

__global__ void axpy_kernel(int n, const double* __restrict__ a, const double* __restrict__ b,
                            double* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = a[i] + b[i];
}

// ---------------------------------------------------------------- PCG
// Device layout of the SIP matrix: structure-of-arrays, entry k of the
// 80 per cell row (slot*16 + col*4 + row) at sip[k*ncell + c]; the block-
// Jacobi inverse likewise at jac[e*ncell + c].

__device__ __forceinline__ void ld4(const double* p, double v[4]) {
  const double2* q = reinterpret_cast<const double2*>(p);
  const double2 a = q[0], b = q[1];
  v[0] = a.x;
  v[1] = a.y;
  v[2] = b.x;
  v[3] = b.y;
}
__device__ __forceinline__ void st4(double* p, const double v[4]) {
  double2* q = reinterpret_cast<double2*>(p);
  q[0] = make_double2(v[0], v[1]);
  q[1] = make_double2(v[2], v[3]);
}

__device__ __forceinline__ void bsr_row(const PcgArgs& a, int c, const double* x, double y[4]) {
  const int ax = c % a.nx, by = c / a.nx;
  const int nb[5] = {c, ax > 0 ? c - 1 : -1, ax + 1 < a.nx ? c + 1 : -1, by > 0 ? c - a.nx : -1,
                     by + 1 < a.ny ? c + a.nx : -1};
  y[0] = y[1] = y[2] = y[3] = 0.0;
#pragma unroll
  for (int s = 0; s < 5; ++s) {
    if (nb[s] < 0) continue;
    double v[4];
    ld4(x + 4 * static_cast<size_t>(nb[s]), v);
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int i = 0; i < 4; ++i) y[i] += a.sip[static_cast<size_t>(s * 16 + j * 4 + i) * a.ncell + c] * v[j];
  }
}

__device__ __forceinline__ void jac_apply(const PcgArgs& a, int c, const double r[4], double z[4]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < 4; ++j) s += a.jac[static_cast<size_t>(j * 4 + i) * a.ncell + c] * r[j];
    z[i] = s;
  }
}

// x = 0, r = b, z = M^-1 r, p = z; partials of r.z and b.b.
__global__ void pcg_init(const PcgArgs a) {
  __shared__ double sh[40];
  double rz = 0.0, bb = 0.0;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < a.ncell; c += gridDim.x * blockDim.x) {
    double r[4], z[4], zero[4] = {0, 0, 0, 0};
    ld4(a.b + 4 * static_cast<size_t>(c), r);
    jac_apply(a, c, r, z);
    st4(a.x + 4 * static_cast<size_t>(c), zero);
    st4(a.r + 4 * static_cast<size_t>(c), r);
    st4(a.z + 4 * static_cast<size_t>(c), z);
    st4(a.p + 4 * static_cast<size_t>(c), z);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      rz += r[i] * z[i];
      bb += r[i] * r[i];
    }
  }
  rz = block_sum(rz, sh);
  if (threadIdx.x == 0) a.part_rz[0 * a.nparts + blockIdx.x] = rz;
  bb = block_sum(bb, sh);
  if (threadIdx.x == 0) a.part_bb[blockIdx.x] = bb;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.state->done = 0;
    a.state->iters = 0;
    a.state->failed = 0;
    a.state->it_base = 0;
  }
}

__global__ void pcg_check_zero(const PcgArgs a) {
  __shared__ double sh[40];
  const double bb = sum_partials(a.part_bb, a.nparts, sh);
  if (threadIdx.x == 0) {
    a.state->bb = bb;
    if (!(bb > 0.0)) a.state->done = 1;  // zero right-hand side: x = 0 exactly
  }
}

// Two adjacent cells of bsr_row at once: the SoA matrix entries of the pair
// as one 16-byte load (ncell even), each cell's neighbours as bsr_row has
// them; per cell the same products in the same order.
__device__ __forceinline__ void bsr_row_pair(const PcgArgs& a, int c, const double* x, double y0[4], double y1[4]) {
  const int ax = c % a.nx, by = c / a.nx;
  const int c1 = c + 1, ax1 = c1 % a.nx, by1 = c1 / a.nx;
  const int nb0[5] = {c, ax > 0 ? c - 1 : -1, ax + 1 < a.nx ? c + 1 : -1, by > 0 ? c - a.nx : -1,
                      by + 1 < a.ny ? c + a.nx : -1};
  const int nb1[5] = {c1, ax1 > 0 ? c1 - 1 : -1, ax1 + 1 < a.nx ? c1 + 1 : -1, by1 > 0 ? c1 - a.nx : -1,
                      by1 + 1 < a.ny ? c1 + a.nx : -1};
#pragma unroll
  for (int i = 0; i < 4; ++i) y0[i] = y1[i] = 0.0;
#pragma unroll
  for (int s = 0; s < 5; ++s) {
    double v0[4] = {0, 0, 0, 0}, v1[4] = {0, 0, 0, 0};
    if (nb0[s] >= 0) ld4(x + 4 * static_cast<size_t>(nb0[s]), v0);
    if (nb1[s] >= 0) ld4(x + 4 * static_cast<size_t>(nb1[s]), v1);
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double2 m = __ldg(reinterpret_cast<const double2*>(a.sip + static_cast<size_t>(s * 16 + j * 4 + i) * a.ncell + c));
        if (nb0[s] >= 0) y0[i] += m.x * v0[j];
        if (nb1[s] >= 0) y1[i] += m.y * v1[j];
      }
  }
}

// q = A p; partials of p.q.  Two cells per thread when ncell is even (16-byte
// matrix loads, twice the bytes in flight per thread).
__global__ void pcg_spmv(const PcgArgs a) {
  if (a.state->done) return;
  __shared__ double sh[40];
  double pq = 0.0;
  if ((a.ncell & 1) == 0) {
    const int npair = a.ncell / 2;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < npair; t += gridDim.x * blockDim.x) {
      const int c = 2 * t;
      double y0[4], y1[4], p0[4], p1[4];
      bsr_row_pair(a, c, a.p, y0, y1);
      st4(a.q + 4 * static_cast<size_t>(c), y0);
      st4(a.q + 4 * static_cast<size_t>(c + 1), y1);
      ld4(a.p + 4 * static_cast<size_t>(c), p0);
      ld4(a.p + 4 * static_cast<size_t>(c + 1), p1);
#pragma unroll
      for (int i = 0; i < 4; ++i) pq += p0[i] * y0[i];
#pragma unroll
      for (int i = 0; i < 4; ++i) pq += p1[i] * y1[i];
    }
  } else {
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < a.ncell; c += gridDim.x * blockDim.x) {
      double y[4], p[4];
      bsr_row(a, c, a.p, y);
      st4(a.q + 4 * static_cast<size_t>(c), y);
      ld4(a.p + 4 * static_cast<size_t>(c), p);
#pragma unroll
      for (int i = 0; i < 4; ++i) pq += p[i] * y[i];
    }
  }
  pq = block_sum(pq, sh);
  if (threadIdx.x == 0) a.part_pq[blockIdx.x] = pq;
}

// alpha = rz/pq; x += alpha p; r -= alpha q; z = M^-1 r; partials r.r, r.z
__global__ void pcg_update(const PcgArgs a, int local) {
  if (a.state->done) return;
  const int it = a.state->it_base + local;
  __shared__ double sh[40];
  const double rz = sum_partials(a.part_rz + (it & 1) * a.nparts, a.nparts, sh);
  const double pq = sum_partials(a.part_pq, a.nparts, sh);
  if (!(pq > 0.0)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      a.state->failed = 1;
      a.state->done = 1;
    }
    return;
  }
  const double alpha = rz / pq;
  double rr = 0.0, rzn = 0.0;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < a.ncell; c += gridDim.x * blockDim.x) {
    const size_t o = 4 * static_cast<size_t>(c);
    double x[4], r[4], p[4], q[4], z[4];
    ld4(a.x + o, x);
    ld4(a.r + o, r);
    ld4(a.p + o, p);
    ld4(a.q + o, q);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      x[i] += alpha * p[i];
      r[i] -= alpha * q[i];
    }
    jac_apply(a, c, r, z);
    st4(a.x + o, x);
    st4(a.r + o, r);
    st4(a.z + o, z);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      rr += r[i] * r[i];
      rzn += r[i] * z[i];
    }
  }
  rr = block_sum(rr, sh);
  if (threadIdx.x == 0) a.part_rr[blockIdx.x] = rr;
  rzn = block_sum(rzn, sh);
  if (threadIdx.x == 0) a.part_rz[((it + 1) & 1) * a.nparts + blockIdx.x] = rzn;
}

// convergence test; beta = rz_new/rz_old; p = z + beta p
__global__ void pcg_direction(const PcgArgs a, int local) {
  if (a.state->done) return;
  const int it = a.state->it_base + local;
  __shared__ double sh[40];
  const double rr = sum_partials(a.part_rr, a.nparts, sh);
  const double bb = a.state->bb;
  if (rr <= a.rtol2 * bb || it + 1 >= a.max_iters) {
    __syncthreads();
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      a.state->done = 1;
      a.state->iters = it + 1;
      a.state->rr = rr;
      if (!(rr <= a.rtol2 * bb)) a.state->failed = 2;
    }
    return;
  }
  const double rz_old = sum_partials(a.part_rz + (it & 1) * a.nparts, a.nparts, sh);
  const double rz_new = sum_partials(a.part_rz + ((it + 1) & 1) * a.nparts, a.nparts, sh);
  const double beta = rz_new / rz_old;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < a.ncell; c += gridDim.x * blockDim.x) {
    const size_t o = 4 * static_cast<size_t>(c);
    double z[4], p[4];
    ld4(a.z + o, z);
    ld4(a.p + o, p);
#pragma unroll
    for (int i = 0; i < 4; ++i) p[i] = z[i] + beta * p[i];
    st4(a.p + o, p);
  }
}

// ---- multigrid-preconditioned variants: the preconditioner application is
// a separate V-cycle between these kernels.
// x = 0, r = b; partials of b.b
__global__ void pcg_init_mg(const PcgArgs a) {
  __shared__ double sh[40];
  double bb = 0.0;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < a.ncell; c += gridDim.x * blockDim.x) {
    double r[4], zero[4] = {0, 0, 0, 0};
    ld4(a.b + 4 * static_cast<size_t>(c), r);
    st4(a.x + 4 * static_cast<size_t>(c), zero);
    st4(a.r + 4 * static_cast<size_t>(c), r);
#pragma unroll
    for (int i = 0; i < 4; ++i) bb += r[i] * r[i];
  }
  bb = block_sum(bb, sh);
  if (threadIdx.x == 0) a.part_bb[blockIdx.x] = bb;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.state->done = 0;
    a.state->iters = 0;
    a.state->failed = 0;
    a.state->it_base = 0;
  }
}
// p = z (init) ; partials of r.z into part_rz[slot], slot = (it_base + local + 1) & 1
// (init: local = -1)
__global__ void pcg_rz(const PcgArgs a, int local, bool copy_p) {
  if (a.state->done) return;
  const int slot = (a.state->it_base + local + 1) & 1;
  __shared__ double sh[40];
  double rz = 0.0;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < a.ncell; c += gridDim.x * blockDim.x) {
    double r[4], z[4];
    ld4(a.r + 4 * static_cast<size_t>(c), r);
    ld4(a.z + 4 * static_cast<size_t>(c), z);
    if (copy_p) st4(a.p + 4 * static_cast<size_t>(c), z);
#pragma unroll
    for (int i = 0; i < 4; ++i) rz += r[i] * z[i];
  }
  rz = block_sum(rz, sh);
  if (threadIdx.x == 0) a.part_rz[slot * a.nparts + blockIdx.x] = rz;
}
// alpha = rz/pq; x += alpha p; r -= alpha q; partials r.r
__global__ void pcg_update_mg(const PcgArgs a, int local) {
  if (a.state->done) return;
  const int it = a.state->it_base + local;
  __shared__ double sh[40];
  const double rz = sum_partials(a.part_rz + (it & 1) * a.nparts, a.nparts, sh);
  const double pq = sum_partials(a.part_pq, a.nparts, sh);
  if (!(pq > 0.0)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      a.state->failed = 1;
      a.state->done = 1;
    }
    return;
  }
  const double alpha = rz / pq;
  double rr = 0.0;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < a.ncell; c += gridDim.x * blockDim.x) {
    const size_t o = 4 * static_cast<size_t>(c);
    double x[4], r[4], p[4], q[4];
    ld4(a.x + o, x);
    ld4(a.r + o, r);
    ld4(a.p + o, p);
    ld4(a.q + o, q);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      x[i] += alpha * p[i];
      r[i] -= alpha * q[i];
      rr += r[i] * r[i];
    }
    st4(a.x + o, x);
    st4(a.r + o, r);
  }
  rr = block_sum(rr, sh);
  if (threadIdx.x == 0) a.part_rr[blockIdx.x] = rr;
}

__global__ void bsr_apply_kernel(const PcgArgs a, const double* x, double* y) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < a.ncell; c += gridDim.x * blockDim.x) {
    double v[4];
    bsr_row(a, c, x, v);
    st4(y + 4 * static_cast<size_t>(c), v);
  }
}

int grid_for(long long n) {
  long long g = (n + kThreads - 1) / kThreads;
  if (g > 148 * 8) g = 148 * 8;
  return static_cast<int>(g < 1 ? 1 : g);
}

}  // namespace

void sigma_apply(int ndof, const double* blocks, const double* x, const double* x_minus,
                 const double* g, double* out, cudaStream_t s) {
  sigma_apply_kernel<<<grid_for(ndof), kThreads, 0, s>>>(ndof, blocks, x, x_minus, g, out);
  RTLR_CUDA(cudaGetLastError());
}

void phi_accumulate(int ndof, int nu, const double* psi, long long ld, const double* w, double* phi,
                    cudaStream_t s) {
  phi_accum_kernel<<<grid_for(ndof), kThreads, 0, s>>>(ndof, nu, psi, ld, w, phi);
  RTLR_CUDA(cudaGetLastError());
}

void diff_norms(int n, const double* a, const double* b, double* work, double* out2, cudaStream_t s) {
  const int parts = kNormParts;
  diff_norm_partials<<<parts, kThreads, 0, s>>>(n, a, b, work, work + parts);
  finish_norms<<<1, kThreads, 0, s>>>(parts, work, work + parts, out2);
  RTLR_CUDA(cudaGetLastError());
}

void vadd(int n, const double* a, const double* b, double* out, cudaStream_t s) {
  axpy_kernel<<<grid_for(n), kThreads, 0, s>>>(n, a, b, out);
  RTLR_CUDA(cudaGetLastError());
}

void bsr_apply(const PcgArgs& a, const double* x, double* y, cudaStream_t s) {
  bsr_apply_kernel<<<grid_for(a.ncell), kThreads, 0, s>>>(a, x, y);
  RTLR_CUDA(cudaGetLastError());
}

namespace {

__global__ void pcg_advance(PcgState* st, int chunk) { st->it_base += chunk; }

bool same_loop(const PcgArgs& u, const PcgArgs& v) {  // everything the loop kernels read (not b)
  return u.nx == v.nx && u.ny == v.ny && u.ncell == v.ncell && u.nparts == v.nparts && u.max_iters == v.max_iters &&
         u.rtol2 == v.rtol2 && u.sip == v.sip && u.jac == v.jac && u.x == v.x && u.r == v.r && u.z == v.z &&
         u.p == v.p && u.q == v.q && u.part_rz == v.part_rz && u.part_pq == v.part_pq && u.part_rr == v.part_rr &&
         u.part_bb == v.part_bb && u.state == v.state && u.mg == v.mg && u.tmp4 == v.tmp4;
}

// One chunk of PCG iterations (every kernel returns at once after state->done).
void pcg_chunk(const PcgArgs& a, int chunk, cudaStream_t s) {
  const int g = a.nparts;
  for (int i = 0; i < chunk; ++i) {
    pcg_spmv<<<g, kThreads, 0, s>>>(a);
    if (a.mg) {
      pcg_update_mg<<<g, kThreads, 0, s>>>(a, i);
      mg_vcycle(a, *a.mg, a.r, a.z, a.tmp4, s);
      pcg_rz<<<g, kThreads, 0, s>>>(a, i, false);
    } else {
      pcg_update<<<g, kThreads, 0, s>>>(a, i);
    }
    pcg_direction<<<g, kThreads, 0, s>>>(a, i);
  }
  pcg_advance<<<1, 1, 0, s>>>(a.state, chunk);
  RTLR_CUDA(cudaGetLastError());
}

}  // namespace

PcgGraph::~PcgGraph() { reset(); }
void PcgGraph::reset() {
  if (exec) cudaGraphExecDestroy(exec);
  exec = nullptr;
}

int pcg_solve(const PcgArgs& a, PcgState* host_state, cudaStream_t s, PcgGraph* graph) {
  const int g = a.nparts;
  if (a.mg) {
    pcg_init_mg<<<g, kThreads, 0, s>>>(a);
    pcg_check_zero<<<1, kThreads, 0, s>>>(a);
    mg_vcycle(a, *a.mg, a.r, a.z, a.tmp4, s);
    pcg_rz<<<g, kThreads, 0, s>>>(a, -1, true);
  } else {
    pcg_init<<<g, kThreads, 0, s>>>(a);
    pcg_check_zero<<<1, kThreads, 0, s>>>(a);
  }
  RTLR_CUDA(cudaGetLastError());
  const int chunk = a.mg ? 8 : 32;
  // The loop body is the same launch sequence every chunk: captured once per
  // buffer set as a CUDA graph (the legacy default stream cannot capture).
  static const bool graphs_off = [] {
    const char* e = std::getenv("RTLR_PCG_GRAPH");
    return e != nullptr && e[0] == '0';
  }();
  const bool use_graph = graph != nullptr && s != nullptr && !graphs_off;
  if (use_graph && (graph->exec == nullptr || graph->chunk != chunk || !same_loop(graph->key, a))) {
    graph->reset();
    cudaGraph_t gr = nullptr;
    RTLR_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    pcg_chunk(a, chunk, s);
    RTLR_CUDA(cudaStreamEndCapture(s, &gr));
    RTLR_CUDA(cudaGraphInstantiate(&graph->exec, gr, 0));
    cudaGraphDestroy(gr);
    graph->key = a;
    graph->chunk = chunk;
  }
  for (int it0 = 0; it0 < a.max_iters; it0 += chunk) {
    if (use_graph)
      RTLR_CUDA(cudaGraphLaunch(graph->exec, s));
    else
      pcg_chunk(a, chunk, s);
    RTLR_CUDA(cudaMemcpyAsync(host_state, a.state, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
    RTLR_CUDA(cudaStreamSynchronize(s));
    if (host_state->done) break;
  }
  if (host_state->failed == 1) throw std::runtime_error("diffusion solve failed");
  return host_state->iters;
}

}  // namespace cuda
}  // namespace rtlr
