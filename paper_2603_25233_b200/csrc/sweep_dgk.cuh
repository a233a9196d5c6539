// General-degree (K != 1) sweep and streaming operator (sweep_dgk.cu).
#pragma once

#include "device.cuh"

namespace rtlr {
namespace cuda {

struct DgkSweepArgs {
  int nx, ny, n;
  const double* dirs;    // N_Omega x 3
  const int* angles;     // n angle indices (nullptr: 0..n-1)
  const double* rhs;     // direction k reads rhs + k * rhs_stride (0: shared)
  long long rhs_stride;
  const double* bc;      // optional per-angle inflow vectors, bc + angle * bc_stride
  long long bc_stride;
  double* psi;           // direction k writes psi + k * psi_stride
  long long psi_stride;
  const double* sigma_t; // ncell x s^2 column-major blocks
  const double* blocks;  // ax-, ax+, ay-, ay+, bx-, bx+, by-, by+ (s x s each)
  int* err;              // set to 1 on a singular local block
};

// sweep(ops, quad, angle, rhs) (sweep.cpp:10-57) for degree K <= 4
void sweep_dgk(int degree, const DgkSweepArgs& a, cudaStream_t s);
// StreamingOperator::apply (operators.cpp:283-288) for degree K <= 4
void apply_dgk(int degree, int nx, int ny, const double* sigma_t, const double* blocks, double omx, double omy,
               const double* v, double* out, cudaStream_t s);

}  // namespace cuda
}  // namespace rtlr
