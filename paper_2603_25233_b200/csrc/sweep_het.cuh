// K1 for heterogeneous media and many directions (sweep_het.cu).
#pragma once

#include "device.cuh"

namespace rtlr {
namespace cuda {

constexpr int kHetD = 4;  // directions per warp

// One launch: ngroups direction groups of kHetD slots, each group one
// quadrant orientation (o = (Omega_x < 0) + 2 (Omega_y < 0)).
struct SweepHetArgs {
  int nx, ny, ngroups, W;
  long long ndof;
  const double* dirs;          // N_Omega x 3
  const int* group_orient;     // ngroups
  const int* slot_angle;       // ngroups x kHetD angle indices (-1: padding)
  const int* slot_pos;         // ngroups x kHetD output columns of psi (-1: none)
  const double* slot_weight;   // ngroups x kHetD scalar-flux weights (nullptr: 0)
  const double* sig_skew;      // skewed Sigma_t (build_skew_layout, 8 planes)
  const double* rhs_skew;      // skewed shared source (build_skew_layout, 2 planes)
  const double* bc;            // optional per-angle inflow, bc + angle * bc_stride (natural layout)
  long long bc_stride;
  double* psi;                 // optional: psi + pos * psi_stride
  long long psi_stride;
  double* phi_part;            // optional: ngroups x ndof scalar-flux partials
  double* line;                // ngroups x W x kHetD x nx x 2 trace lines
  int* err;
  StreamDev sc;
};

// Skewed copies of a per-cell field (planes x 16 bytes per cell) for the
// four orientations: out[o][band][d][plane][lane] holds cell (row band*32 +
// lane, col d - lane) in that orientation's sweep order (zero padding).
size_t skew_layout_doubles(int nx, int ny, int planes);
void build_skew_layout(int nx, int ny, const double* cells, int planes, double* out, cudaStream_t s);
// warps per direction group for a launch of ngroups groups
int sweep_het_warps(int nx, int ny, int ngroups);
void launch_sweep_het(const SweepHetArgs& a, cudaStream_t s);
// phi = sum_g part[g] (fixed order)
void reduce_phi_parts(long long ndof, int groups, const double* part, double* phi, cudaStream_t s);

}  // namespace cuda
}  // namespace rtlr
