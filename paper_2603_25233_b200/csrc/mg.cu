// Multigrid V-cycle preconditioner for the SIP-DG DSA system (see mg.cuh).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <stdexcept>

#include "linalg.cuh"
#include "mg.cuh"

namespace rtlr {
namespace cuda {

namespace {

constexpr double kOmegaDG = 0.7;   // damped block-Jacobi on the SIP-DG level
constexpr double kOmega5 = 0.8;    // damped Jacobi on the 5-point levels

int grid_for(long long n) {
  long long g = (n + 255) / 256;
  return static_cast<int>(std::max<long long>(1, std::min<long long>(g, 148 * 8)));
}

// ---------------------------------------------------------------- DG level
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
__device__ __forceinline__ void jac(const PcgArgs& a, int c, const double r[4], double z[4]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < 4; ++j) s += a.jac[static_cast<size_t>(j * 4 + i) * a.ncell + c] * r[j];
    z[i] = s;
  }
}

// x = omega J^-1 b
__global__ void dg_first(const PcgArgs a, const double* __restrict__ b, double* __restrict__ x) {
  if (a.state->done) return;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < a.ncell; c += gridDim.x * blockDim.x) {
    double r[4], z[4];
    ld4(b + 4 * static_cast<size_t>(c), r);
    jac(a, c, r, z);
#pragma unroll
    for (int i = 0; i < 4; ++i) z[i] *= kOmegaDG;
    st4(x + 4 * static_cast<size_t>(c), z);
  }
}
// xo = x + omega J^-1 (b - A x)
__global__ void dg_smooth(const PcgArgs a, const double* __restrict__ b, const double* __restrict__ x,
                          double* __restrict__ xo) {
  if (a.state->done) return;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < a.ncell; c += gridDim.x * blockDim.x) {
    double ax[4], bb[4], xx[4], z[4];
    bsr_row(a, c, x, ax);
    ld4(b + 4 * static_cast<size_t>(c), bb);
    ld4(x + 4 * static_cast<size_t>(c), xx);
#pragma unroll
    for (int i = 0; i < 4; ++i) bb[i] -= ax[i];
    jac(a, c, bb, z);
#pragma unroll
    for (int i = 0; i < 4; ++i) xx[i] += kOmegaDG * z[i];
    st4(xo + 4 * static_cast<size_t>(c), xx);
  }
}
// r1[c] = (b - A x)[4c]   (P0 restriction: the cell-average mode)
__global__ void dg_restrict(const PcgArgs a, const double* __restrict__ b, const double* __restrict__ x,
                            double* __restrict__ r1) {
  if (a.state->done) return;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < a.ncell; c += gridDim.x * blockDim.x) {
    double ax[4];
    bsr_row(a, c, x, ax);
    r1[c] = b[4 * static_cast<size_t>(c)] - ax[0];
  }
}
__global__ void dg_prolong(const PcgArgs a, double* __restrict__ x, const double* __restrict__ x1) {
  if (a.state->done) return;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < a.ncell; c += gridDim.x * blockDim.x)
    x[4 * static_cast<size_t>(c)] += x1[c];
}

// ---------------------------------------------------------------- 5-point levels
struct L5 {
  int nx, ny, n;
  const double* st;  // diag, W, E, S, N (SoA)
};
__device__ __forceinline__ double ax5(const L5& L, int c, const double* x) {
  const int a = c % L.nx, b = c / L.nx;
  double s = L.st[c] * x[c];
  if (a > 0) s += L.st[L.n + c] * x[c - 1];
  if (a + 1 < L.nx) s += L.st[2 * L.n + c] * x[c + 1];
  if (b > 0) s += L.st[3 * L.n + c] * x[c - L.nx];
  if (b + 1 < L.ny) s += L.st[4 * L.n + c] * x[c + L.nx];
  return s;
}
__global__ void l5_first(const int* done, const L5 L, const double* __restrict__ b, double* __restrict__ x) {
  if (*done) return;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < L.n; c += gridDim.x * blockDim.x)
    x[c] = kOmega5 * b[c] / L.st[c];
}
__global__ void l5_smooth(const int* done, const L5 L, const double* __restrict__ b, const double* __restrict__ x,
                          double* __restrict__ xo) {
  if (*done) return;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < L.n; c += gridDim.x * blockDim.x)
    xo[c] = x[c] + kOmega5 * (b[c] - ax5(L, c, x)) / L.st[c];
}
// coarse residual: sum over the (<= 4) children of (b - A x)
__global__ void l5_restrict(const int* done, const L5 L, const double* __restrict__ b, const double* __restrict__ x,
                            int cnx, int cny, double* __restrict__ rc) {
  if (*done) return;
  for (int C = blockIdx.x * blockDim.x + threadIdx.x; C < cnx * cny; C += gridDim.x * blockDim.x) {
    const int A = C % cnx, B = C / cnx;
    double s = 0.0;
    for (int db = 0; db < 2; ++db)
      for (int da = 0; da < 2; ++da) {
        const int a = 2 * A + da, bb = 2 * B + db;
        if (a < L.nx && bb < L.ny) {
          const int f = bb * L.nx + a;
          s += b[f] - ax5(L, f, x);
        }
      }
    rc[C] = s;
  }
}
__global__ void l5_prolong(const int* done, const L5 L, double* __restrict__ x, const double* __restrict__ xc, int cnx) {
  if (*done) return;
  for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < L.n; f += gridDim.x * blockDim.x) {
    const int a = f % L.nx, b = f / L.nx;
    x[f] += xc[(b / 2) * cnx + a / 2];
  }
}
__global__ void dense_apply(const int* done, int n, const double* __restrict__ inv, const double* __restrict__ b,
                            double* __restrict__ x) {
  if (*done) return;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < n; ++j) s += inv[i + j * n] * b[j];
    x[i] = s;
  }
}

// Cycle shape.  Defaults were chosen by measuring PCG iterations and DSA
// time on C1-C4 (K12); the environment overrides exist for that
// tuning only.
struct MgKnobs {
  int nu5 = 2;        // damped-Jacobi steps before and after the coarse correction, 5-point levels
  int nu_dg = 1;      // block-Jacobi steps before and after, DG level
  int w_levels = 0;   // the first w_levels 5-point levels recurse twice (W-cycle)
  // Aggregated operators scaled by 1/alpha.  The Galerkin product of 2x2
  // piecewise-constant aggregation doubles every face coupling relative to a
  // re-discretisation on the coarse grid, so the plain coarse correction
  // under-corrects smooth error; alpha ~2 restores it (C4: 344 -> 78 PCG
  // iterations per DSA solve).  Still an SPD preconditioner: symmetric
  // cycle, A-convergent smoothers, SPD coarse operators.
  double alpha = 2.2;
};
const MgKnobs& knobs() {
  static const MgKnobs k = [] {
    MgKnobs v;
    if (const char* e = std::getenv("RTLR_MG_NU5")) v.nu5 = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("RTLR_MG_NUDG")) v.nu_dg = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("RTLR_MG_WLEVELS")) v.w_levels = std::max(0, std::atoi(e));
    if (const char* e = std::getenv("RTLR_MG_ALPHA")) v.alpha = std::atof(e);
    if (!(v.alpha > 0.0)) v.alpha = 2.2;
    return v;
  }();
  return k;
}

// x[l] <- one cycle for A_l x = b[l], from x = 0 (zero) or from the x[l] held.
// The coarse end of the V-cycle (every 5-point level from l0 down, and the
// dense coarsest solve) in one CTA: the same smooth / restrict / prolong /
// dense steps as the per-level launches, in the same order and with the
// same arithmetic per element, separated by block barriers instead of
// kernel boundaries.  On the small levels the launches were pure latency.
constexpr int kMaxLev = 24;
constexpr int kFuseCells = 64 * 64;  // levels at or below this size run fused
struct CoarseView {
  int l0, nlev, nu5, ncoarse;
  int nx[kMaxLev], ny[kMaxLev];
  const double* st[kMaxLev];
  double *x[kMaxLev], *b[kMaxLev], *t[kMaxLev];
  const double* cinv;
};

__global__ void __launch_bounds__(1024) coarse_cycle(const int* done, const CoarseView v) {
  if (*done) return;
  const int tid = threadIdx.x, nt = blockDim.x;
  double* cur[kMaxLev];
  double* oth[kMaxLev];
  // descent: pre-smoothing from zero, restriction
  for (int l = v.l0; l < v.nlev - 1; ++l) {
    const L5 L{v.nx[l], v.ny[l], v.nx[l] * v.ny[l], v.st[l]};
    double* c = v.x[l];
    double* o = v.t[l];
    for (int i = tid; i < L.n; i += nt) c[i] = kOmega5 * v.b[l][i] / L.st[i];
    __syncthreads();
    for (int it = 1; it < v.nu5; ++it) {
      for (int i = tid; i < L.n; i += nt) o[i] = c[i] + kOmega5 * (v.b[l][i] - ax5(L, i, c)) / L.st[i];
      __syncthreads();
      double* tt = c;
      c = o;
      o = tt;
    }
    const int cnx = v.nx[l + 1], cny = v.ny[l + 1];
    for (int C = tid; C < cnx * cny; C += nt) {
      const int A = C % cnx, B = C / cnx;
      double sum = 0.0;
      for (int db = 0; db < 2; ++db)
        for (int da = 0; da < 2; ++da) {
          const int a = 2 * A + da, bb = 2 * B + db;
          if (a < L.nx && bb < L.ny) {
            const int f = bb * L.nx + a;
            sum += v.b[l][f] - ax5(L, f, c);
          }
        }
      v.b[l + 1][C] = sum;
    }
    __syncthreads();
    cur[l] = c;
    oth[l] = o;
  }
  // coarsest: x = inv b
  {
    const int l = v.nlev - 1, n = v.ncoarse;
    for (int i = tid; i < n; i += nt) {
      double sum = 0.0;
      for (int j = 0; j < n; ++j) sum += v.cinv[i + j * n] * v.b[l][j];
      v.x[l][i] = sum;
    }
    __syncthreads();
  }
  // ascent: prolongation, post-smoothing, result into x[l]
  for (int l = v.nlev - 2; l >= v.l0; --l) {
    const L5 L{v.nx[l], v.ny[l], v.nx[l] * v.ny[l], v.st[l]};
    double* c = cur[l];
    double* o = oth[l];
    const int cnx = v.nx[l + 1];
    for (int f = tid; f < L.n; f += nt) {
      const int a = f % L.nx, bb = f / L.nx;
      c[f] += v.x[l + 1][(bb / 2) * cnx + a / 2];
    }
    __syncthreads();
    for (int it = 0; it < v.nu5; ++it) {
      for (int i = tid; i < L.n; i += nt) o[i] = c[i] + kOmega5 * (v.b[l][i] - ax5(L, i, c)) / L.st[i];
      __syncthreads();
      double* tt = c;
      c = o;
      o = tt;
    }
    if (c != v.x[l]) {
      for (int i = tid; i < L.n; i += nt) v.x[l][i] = c[i];
      __syncthreads();
    }
  }
}

void cycle5(const int* done, const MgDevice& mg, int l, bool zero, cudaStream_t s) {
  {
    const MgKnobs& kk = knobs();
    static const bool fuse_off = [] {  // RTLR_MG_FUSE=0: one launch per step on every level
      const char* e = std::getenv("RTLR_MG_FUSE");
      return e && e[0] == '0';
    }();
    if (!fuse_off && zero && l < mg.nlev - 1 && static_cast<long long>(mg.nx[l]) * mg.ny[l] <= kFuseCells &&
        l >= kk.w_levels && mg.nlev <= kMaxLev) {
      CoarseView v{};
      v.l0 = l;
      v.nlev = mg.nlev;
      v.nu5 = kk.nu5;
      v.ncoarse = mg.ncoarse;
      v.cinv = mg.cinv;
      for (int q = 0; q < mg.nlev; ++q) {
        v.nx[q] = mg.nx[q];
        v.ny[q] = mg.ny[q];
        v.st[q] = mg.st[q];
        v.x[q] = mg.x[q];
        v.b[q] = mg.b[q];
        v.t[q] = mg.t[q];
      }
      coarse_cycle<<<1, 1024, 0, s>>>(done, v);
      return;
    }
  }
  if (l == mg.nlev - 1) {
    if (!zero) throw std::logic_error("multigrid: second visit of the coarsest level");
    dense_apply<<<1, 256, 0, s>>>(done, mg.ncoarse, mg.cinv, mg.b[l], mg.x[l]);
    return;
  }
  const MgKnobs& k = knobs();
  const L5 L{mg.nx[l], mg.ny[l], mg.nx[l] * mg.ny[l], mg.st[l]};
  const int g = grid_for(L.n);
  double* cur = mg.x[l];
  double* oth = mg.t[l];
  int i = 0;
  if (zero) {
    l5_first<<<g, 256, 0, s>>>(done, L, mg.b[l], cur);
    i = 1;
  }
  for (; i < k.nu5; ++i) {
    l5_smooth<<<g, 256, 0, s>>>(done, L, mg.b[l], cur, oth);
    std::swap(cur, oth);
  }
  const int cnx = mg.nx[l + 1], cny = mg.ny[l + 1];
  l5_restrict<<<grid_for(static_cast<long long>(cnx) * cny), 256, 0, s>>>(done, L, mg.b[l], cur, cnx, cny,
                                                                          mg.b[l + 1]);
  cycle5(done, mg, l + 1, true, s);
  if (l < k.w_levels && l + 1 < mg.nlev - 1) cycle5(done, mg, l + 1, false, s);
  l5_prolong<<<g, 256, 0, s>>>(done, L, cur, mg.x[l + 1], cnx);
  for (i = 0; i < k.nu5; ++i) {
    l5_smooth<<<g, 256, 0, s>>>(done, L, mg.b[l], cur, oth);
    std::swap(cur, oth);
  }
  if (cur != mg.x[l])
    RTLR_CUDA(cudaMemcpyAsync(mg.x[l], cur, L.n * sizeof(double), cudaMemcpyDeviceToDevice, s));
}

void invert_dense(int n, std::vector<double>& a) {  // Gauss-Jordan, partial pivoting, column-major
  std::vector<double> inv(static_cast<size_t>(n) * n, 0.0);
  for (int i = 0; i < n; ++i) inv[i + static_cast<size_t>(i) * n] = 1.0;
  for (int k = 0; k < n; ++k) {
    int p = k;
    for (int i = k + 1; i < n; ++i)
      if (std::abs(a[i + static_cast<size_t>(k) * n]) > std::abs(a[p + static_cast<size_t>(k) * n])) p = i;
    if (a[p + static_cast<size_t>(k) * n] == 0.0) throw std::runtime_error("multigrid: singular coarsest operator");
    for (int j = 0; j < n; ++j) {
      std::swap(a[k + static_cast<size_t>(j) * n], a[p + static_cast<size_t>(j) * n]);
      std::swap(inv[k + static_cast<size_t>(j) * n], inv[p + static_cast<size_t>(j) * n]);
    }
    const double d = a[k + static_cast<size_t>(k) * n];
    for (int j = 0; j < n; ++j) {
      a[k + static_cast<size_t>(j) * n] /= d;
      inv[k + static_cast<size_t>(j) * n] /= d;
    }
    for (int i = 0; i < n; ++i) {
      if (i == k) continue;
      const double f = a[i + static_cast<size_t>(k) * n];
      if (f == 0.0) continue;
      for (int j = 0; j < n; ++j) {
        a[i + static_cast<size_t>(j) * n] -= f * a[k + static_cast<size_t>(j) * n];
        inv[i + static_cast<size_t>(j) * n] -= f * inv[k + static_cast<size_t>(j) * n];
      }
    }
  }
  a.swap(inv);
}

}  // namespace

std::vector<MgLevelHost> build_mg_hierarchy(int nx, int ny, const std::vector<double>& sip, int coarsest_cells,
                                            std::vector<double>& coarse_inv) {
  std::vector<MgLevelHost> lv;
  MgLevelHost l0{nx, ny, {}};
  const size_t n0 = static_cast<size_t>(nx) * ny;
  l0.st.assign(5 * n0, 0.0);
  for (size_t c = 0; c < n0; ++c)
    for (int s = 0; s < 5; ++s) l0.st[s * n0 + c] = sip[(c * 5 + s) * 16];  // entry (0,0): P0^T A P0
  lv.push_back(std::move(l0));
  while (static_cast<long long>(lv.back().nx) * lv.back().ny > coarsest_cells && (lv.back().nx > 1 || lv.back().ny > 1)) {
    const MgLevelHost& f = lv.back();
    const int cnx = (f.nx + 1) / 2, cny = (f.ny + 1) / 2;
    const size_t nf = static_cast<size_t>(f.nx) * f.ny, nc = static_cast<size_t>(cnx) * cny;
    MgLevelHost c{cnx, cny, std::vector<double>(5 * nc, 0.0)};
    for (int b = 0; b < f.ny; ++b)
      for (int a = 0; a < f.nx; ++a) {
        const size_t fi = static_cast<size_t>(b) * f.nx + a;
        const int A = a / 2, B = b / 2;
        const size_t C = static_cast<size_t>(B) * cnx + A;
        c.st[C] += f.st[fi];
        const int na[4] = {a - 1, a + 1, a, a};
        const int nbb[4] = {b, b, b - 1, b + 1};
        for (int d = 0; d < 4; ++d) {
          if (na[d] < 0 || na[d] >= f.nx || nbb[d] < 0 || nbb[d] >= f.ny) continue;
          const double v = f.st[(d + 1) * nf + fi];
          const int GA = na[d] / 2, GB = nbb[d] / 2;
          if (GA == A && GB == B)
            c.st[C] += v;  // coupling inside the aggregate
          else
            c.st[(d + 1) * nc + C] += v;  // same direction between aggregates
        }
      }
    if (knobs().alpha != 1.0)
      for (double& v : c.st) v /= knobs().alpha;
    lv.push_back(std::move(c));
  }
  // dense inverse of the coarsest level
  const MgLevelHost& L = lv.back();
  const int n = L.nx * L.ny;
  std::vector<double> a(static_cast<size_t>(n) * n, 0.0);
  for (int b = 0; b < L.ny; ++b)
    for (int x = 0; x < L.nx; ++x) {
      const int c = b * L.nx + x;
      a[c + static_cast<size_t>(c) * n] = L.st[c];
      if (x > 0) a[c + static_cast<size_t>(c - 1) * n] = L.st[n + c];
      if (x + 1 < L.nx) a[c + static_cast<size_t>(c + 1) * n] = L.st[2 * n + c];
      if (b > 0) a[c + static_cast<size_t>(c - L.nx) * n] = L.st[3 * n + c];
      if (b + 1 < L.ny) a[c + static_cast<size_t>(c + L.nx) * n] = L.st[4 * n + c];
    }
  invert_dense(n, a);
  coarse_inv = std::move(a);
  return lv;
}

void mg_vcycle(const PcgArgs& a, const MgDevice& mg, const double* r, double* z, double* tmp4, cudaStream_t s) {
  const int g = grid_for(a.ncell);
  const int* done = &a.state->done;
  const MgKnobs& k = knobs();
  const size_t bytes = 4 * static_cast<size_t>(a.ncell) * sizeof(double);
  // pre-smooth from zero: z = omega J^-1 r, then nu_dg - 1 more steps
  double* cur = z;
  double* oth = tmp4;
  dg_first<<<g, 256, 0, s>>>(a, r, cur);
  for (int i = 1; i < k.nu_dg; ++i) {
    dg_smooth<<<g, 256, 0, s>>>(a, r, cur, oth);
    std::swap(cur, oth);
  }
  // coarse correction through the cell-average level
  dg_restrict<<<g, 256, 0, s>>>(a, r, cur, mg.b[0]);
  cycle5(done, mg, 0, true, s);
  dg_prolong<<<g, 256, 0, s>>>(a, cur, mg.x[0]);
  // post-smooth (same damped block Jacobi)
  for (int i = 0; i < k.nu_dg; ++i) {
    dg_smooth<<<g, 256, 0, s>>>(a, r, cur, oth);
    std::swap(cur, oth);
  }
  if (cur != z) RTLR_CUDA(cudaMemcpyAsync(z, cur, bytes, cudaMemcpyDeviceToDevice, s));
  RTLR_CUDA(cudaGetLastError());
}

}  // namespace cuda
}  // namespace rtlr
