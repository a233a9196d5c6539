// Multigrid V-cycle preconditioner for the DSA's SIP-DG system (K12,
// SURVEY.md §8(f)1): block-Jacobi smoothing on the DG level, a cell-average
// (P0) level whose operator is the Galerkin product P0^T A P0 (entry (0,0)
// of every 4x4 BSR block: a 5-point stencil), then 2x2 aggregation levels
// with scaled Galerkin coarse operators (again 5-point; see MgKnobs::alpha)
// down to a small grid solved by a dense inverse.  Symmetric (equal pre/post damped Jacobi), so
// it is a valid CG preconditioner.  Deterministic: no atomics.
#pragma once

#include <vector>

#include "device.cuh"

namespace rtlr {
namespace cuda {

struct MgLevelHost {
  int nx, ny;
  std::vector<double> st;  // 5 x ncell (diag, W, E, S, N), structure-of-arrays
};

// Builds the P0 + aggregation hierarchy on the host from the BSR SIP matrix
// (ncell x 5 x 16, block column-major; slot order self, W, E, S, N).
std::vector<MgLevelHost> build_mg_hierarchy(int nx, int ny, const std::vector<double>& sip_bsr,
                                            int coarsest_cells, std::vector<double>& coarse_inv);

struct MgDevice {
  int nlev = 0;                 // aggregation levels incl. the P0 level
  std::vector<int> nx, ny;
  std::vector<double*> st;      // 5 x ncell per level
  std::vector<double*> x, b, t; // per-level vectors
  double* cinv = nullptr;       // dense inverse of the coarsest level
  int ncoarse = 0;
};

struct PcgArgs;
// z = M^-1 r with one V-cycle; skipped when state->done is set.
void mg_vcycle(const PcgArgs& a, const MgDevice& mg, const double* r, double* z, double* tmp4, cudaStream_t s);

}  // namespace cuda
}  // namespace rtlr
