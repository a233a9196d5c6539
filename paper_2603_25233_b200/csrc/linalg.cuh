// Vector / DSA kernels (see linalg.cu).
#pragma once

#include "device.cuh"

namespace rtlr {
namespace cuda {

constexpr int kNormParts = 296;  // 2 x 148 SMs

struct PcgState {
  double bb, rr;
  int done, iters, failed, it_base;  // it_base: first iteration of the running chunk
};

struct PcgArgs {
  int nx, ny, ncell, nparts, max_iters;
  double rtol2;
  const double* sip;  // SoA, 80 x ncell
  const double* jac;  // SoA, 16 x ncell
  const double* b;
  double *x, *r, *z, *p, *q;
  double *part_rz, *part_pq, *part_rr, *part_bb;  // part_rz has 2 x nparts
  PcgState* state;
  const struct MgDevice* mg = nullptr;  // multigrid preconditioner (nullptr: block Jacobi)
  double* tmp4 = nullptr;               // N_x scratch for the V-cycle
};

// out = Sigma (x - x_minus) + g   (x_minus, g optional)
void sigma_apply(int ndof, const double* blocks, const double* x, const double* x_minus,
                 const double* g, double* out, cudaStream_t s);
void phi_accumulate(int ndof, int nu, const double* psi, long long ld, const double* w, double* phi,
                    cudaStream_t s);
// out2[0] = ||a-b||_2, out2[1] = ||a-b||_inf (b optional); work >= 2*kNormParts
void diff_norms(int n, const double* a, const double* b, double* work, double* out2, cudaStream_t s);
void vadd(int n, const double* a, const double* b, double* out, cudaStream_t s);
void bsr_apply(const PcgArgs& a, const double* x, double* y, cudaStream_t s);
// Cached CUDA graph of one chunk of PCG iterations (pcg_solve); rebuilt when
// the loop's buffers change.
struct PcgGraph {
  cudaGraphExec_t exec = nullptr;
  PcgArgs key{};
  int chunk = 0;
  PcgGraph() = default;
  PcgGraph(const PcgGraph&) = delete;
  PcgGraph& operator=(const PcgGraph&) = delete;
  ~PcgGraph();
  void reset();
};
int pcg_solve(const PcgArgs& a, PcgState* host_state, cudaStream_t s, PcgGraph* graph = nullptr);

}  // namespace cuda
}  // namespace rtlr
