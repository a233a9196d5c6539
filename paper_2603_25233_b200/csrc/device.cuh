// Device-side declarations for the B200 compute core (sm_100a).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>

namespace rtlr {
namespace cuda {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define RTLR_CUDA(call)                                                                 \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      throw ::rtlr::cuda::CudaError(std::string("CUDA error ") + cudaGetErrorString(e_) + \
                                    " at " + __FILE__ + ":" + std::to_string(__LINE__)); \
  } while (0)

// Per-problem constants the kernels read (K = 1).
struct StreamDev {
  double ax_minus[16], ax_plus[16], ay_minus[16], ay_plus[16];
  double bx_minus[16], bx_plus[16], by_minus[16], by_plus[16];
  double trx_r[2], trx_l[2], try_r[2], try_l[2];
};

// Geometry + operator data for the streaming stencil (StreamingOperator).
struct StencilArgs {
  int nx, ny, ncell;
  const double* sigma_t;  // ncell x 16
  StreamDev sc;
};

// out = (Sigma_t + omx D_x^{+-} + omy D_y^{+-}) v   (operators.cpp:283-288)
void launch_stream_apply(const StencilArgs& a, double omx, double omy, const double* v, double* out,
                         cudaStream_t s);
// norms[k] = || rhs (+ bc_k) - A_k y_k ||_2 for a batch of m angles, y_k =
// Y + k*ldy.  Deterministic: fixed per-angle reduction tree independent of
// the batch position.  work >= m * residual_parts(ncell) doubles.
int residual_parts(int ncell);
void launch_residual_norms(const StencilArgs& a, int m, const int* d_angles, const double* d_dirs,
                           const double* Y, long long ldy, const double* rhs, const double* bc,
                           long long bc_stride, double* work, double* norms, cudaStream_t s);

// One batched sweep launch: n directions, one warp each.
struct SweepArgs {
  int nx, ny, n;
  const double* dirs;       // [N_Omega x 3] (omega_x, omega_y, omega_z)
  const int* angles;        // n angle indices into dirs (nullptr: 0..n-1)
  const double* rhs;        // base; direction k reads rhs + k*rhs_stride
  long long rhs_stride;     // 0 = shared right-hand side
  const double* bc;         // optional per-angle inflow: bc + angle*bc_stride
  long long bc_stride;
  double* psi;              // direction k writes psi + k*psi_stride
  long long psi_stride;
  const double* sigma_t;    // ncell x 16 blocks (general path) / 16 (uniform)
  double* line;             // n x nx x 2 inter-band trace buffers
  int* err;                 // set to 1 on a singular local block
  StreamDev sc;
  // Optional (general media, row-scan kernel): per-direction per-cell block
  // data factored ahead of the sweep, n x kPrefDoubles x pref_stride
  // (structure of arrays; see launch_sweep_prefactor).
  const double* pref = nullptr;
  long long pref_stride = 0;
  // Wide kernel: psi leaves through the consumed source tile (shared memory):
  // 2 one TMA store per whole chunk, 1 a coalesced read-back with 1 KB
  // contiguous per store instruction, 0 the lanes' own 128-byte runs (set by
  // the launcher, RTLR_SCAN_STOUT).
  int stage_out = 0;
};

// Per (direction, cell): M^-1 (16, column-major), Qc = -M^-1 K_x (8), G = T_x Qc (4)
// for M = Omega_x A_x + Omega_y A_y + Sigma_t(cell), factored with the
// reference's partial-pivot LU and singular test.  Off the sweep's critical
// path, so latency-bound sweeps (a few directions, heterogeneous media) step
// faster.  table: n x kPrefDoubles x stride doubles; stride >= ncell, even.
constexpr int kPrefDoubles = 28;
constexpr int kPrefMinvDoubles = 16;  // M^-1 only (the wavefront kernel's table)
void launch_sweep_prefactor(const SweepArgs& a, double* table, long long stride, cudaStream_t s,
                            int planes = kPrefDoubles);

// Skewed lane-per-row wavefront (sweep.cu) and row-chunk affine-scan
// (sweep_scan.cu) formulations of K1; Problem::sweep picks the scan kernel
// unless RTLR_SWEEP=skew.
void launch_sweep(const SweepArgs& a, bool uniform_sigma_t, cudaStream_t s);
void launch_sweep_scan(const SweepArgs& a, bool uniform_sigma_t, cudaStream_t s);
// Few-direction wavefront sweep: one thread-block cluster (cluster CTAs x 8
// warps) per direction, rows interleaved over the cluster's warps, traces
// handed on through distributed shared memory.  General media need a.pref
// (kPrefMinvDoubles planes).  cluster 0: sweep_wave_cluster's choice.
void launch_sweep_wave(const SweepArgs& a, bool uniform_sigma_t, int cluster, cudaStream_t s);
// Cluster size for the wavefront kernel on this launch (all n clusters
// co-resident), or 0 when it does not apply (too many directions, rows too
// wide for the shared-memory trace lines).
int sweep_wave_cluster(const SweepArgs& a, bool uniform_sigma_t);

// Generates C5 sources: rhs[k][dof] = U[0,1)(seed, (dir0+k)*ndof + dof).
void launch_c5_fill(double* rhs, long long n_dirs, long long dir0, long long ndof,
                    std::uint64_t seed, cudaStream_t s);

}  // namespace cuda
}  // namespace rtlr
