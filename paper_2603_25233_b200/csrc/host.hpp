// Host-side setup for the B200 compute core of rtlr (arXiv 2603.25233).
//
// Everything here runs once per problem on the host and produces the arrays
// the device kernels consume.  The arithmetic follows the reference
// expression by expression so the inputs are bitwise identical to what the
// reference's solver sees (quadrature, cell indexing, cross-section blocks,
// source projection, SIP-DG diffusion matrix); tests/ check this against
// the oracle restatement.  The solvers run DG degree K = 1 (s = 4 DOFs per
// cell); K = 0 and 2..4 assemble for the sweep and the streaming operator
// (host_dgk.cpp).
#pragma once

#include <cstdint>
#include <functional>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

namespace rtlr {
namespace cuda {

using Field = std::function<double(double, double)>;  // ScalarField (dg_space.hpp:10)

struct ConfigError : std::runtime_error {  // problem.hpp:16-18
  using std::runtime_error::runtime_error;
};

// proj/include/rtlr/problem.hpp:54-67
struct SolverParams {
  double eps_si_sa = 1e-6, eps_res = 1e-7, eps_diff = 1e-7, eps_svd = 1e-8, eps_mgs = 1e-10;
  int p = 1, q = 8;
  std::uint64_t seed = 0;
  int max_iterations = 500;
  bool use_dsa = true, store_psi = true, build_factors = true;
};

// proj/include/rtlr/problem.hpp:69-81 with fields as callables.
struct ProblemConfig {
  std::string preset;
  double x_min = -1, x_max = 1, y_min = -1, y_max = 1;
  int nx = 32, ny = 32, n_theta = 16, n_omega_z = 8, degree = 1;
  Field sigma_s, sigma_a, source, boundary;
  bool boundary_zero = true;
  SolverParams solver;
};

// Presets of proj/src/problem.cpp:111-200 ("homogeneous(s,L)",
// "variable_scattering", "pin_cell", "lattice", suffix ":full") and the
// BASELINE configs "C1".."C5".
ProblemConfig make_config(const std::string& name);
void validate_config(const ProblemConfig& c);  // problem.cpp:95-107

// proj/src/quadrature.cpp
double legendre_value(int n, double x);
double legendre_derivative(int n, double x);
void gauss_legendre(int n, std::vector<double>& nodes, std::vector<double>& weights);
void build_cl_quadrature(int n_theta, int n_omega_z, std::vector<double>& dirs,
                         std::vector<double>& weights);

// Streaming constants for K = 1 (proj/src/operators.cpp:13-79), all in the
// reference's arithmetic: 4x4 diagonal blocks column-major, traces.
struct StreamConsts {
  double ax_minus[16], ax_plus[16], ay_minus[16], ay_plus[16];
  double bx_minus[16], bx_plus[16], by_minus[16], by_plus[16];
  double trx_r[2], trx_l[2], try_r[2], try_l[2];
};

// Assembled problem on the host (AssembledProblem, problem.hpp:98-106).
struct HostProblem {
  ProblemConfig cfg;
  int nx = 0, ny = 0, ncell = 0, ndof = 0, n_omega = 0;
  double dx = 0, dy = 0;
  std::vector<double> dirs, weights;              // N_Omega x 3 row-major, N_Omega
  std::vector<double> sigma_t, sigma_s, sigma_a;  // ncell x 16, block column-major
  std::vector<double> source;                     // N_x
  bool bc_any = false;
  std::vector<double> bc;                         // N_Omega x N_x when bc_any
  StreamConsts sc;
  // SIP-DG diffusion matrix (+ Sigma_a) in cell-blocked BSR: 5 blocks per
  // cell row in the order self, west (a-1), east (a+1), south (b-1),
  // north (b+1); each 4x4 column-major; absent neighbours are zero blocks.
  std::vector<double> sip;  // ncell x 5 x 16
  bool sigma_t_uniform = false;  // every sigma_t block bitwise identical
  double assembly_seconds = 0.0;
  // DG degree K and DOFs per cell s = (K+1)^2.  K != 1 (host_dgk.cpp): the
  // sigma blocks are ncell x s^2 and kblocks holds the streaming blocks
  // ax-, ax+, ay-, ay+, bx-, bx+, by-, by+ (s x s column-major each); only
  // the sweep and the streaming operator run on such a problem.
  int degree = 1, spc = 4;
  std::vector<double> kblocks;
};

constexpr int kMaxDegree = 4;  // K <= 4 (s <= 25) on the GPU path
// Assembly for DG degree K != 1 (operators.cpp:13-281 for any K).
void assemble_general(const ProblemConfig& cfg, HostProblem& out);
void boundary_vector_general(const HostProblem& hp, const Field& g, int angle, double* out);

void assemble(const ProblemConfig& cfg, HostProblem& out);

// A caller-assembled problem (the inputs of solve_full_rank(ops, quad, bc,
// source, dsa, ...), full_rank.hpp:41-43, as plain arrays): the K = 1 mesh,
// any direction set, per-cell 4x4 cross-section blocks (column-major),
// the projected source, optional per-angle inflow vectors and optional SIP
// matrix.  Pointers are borrowed for the call.
struct ProblemArrays {
  int nx = 0, ny = 0;
  double x_min = 0, x_max = 1, y_min = 0, y_max = 1;
  int n_theta = 0, n_omega_z = 0;  // CL shape (0, 0: unstructured; n_omega given)
  int n_omega = 0;
  const double* dirs = nullptr;      // n_omega x 3 row-major
  const double* weights = nullptr;   // n_omega
  const double* sigma_t = nullptr;   // ncell x 16
  const double* sigma_s = nullptr;   // ncell x 16
  const double* sigma_a = nullptr;   // ncell x 16 or null (= sigma_t - sigma_s)
  const double* source = nullptr;    // N_x
  const double* boundary = nullptr;  // n_omega x N_x or null (vacuum)
  const double* sip = nullptr;       // ncell x 5 x 16 or null (built from the blocks when use_dsa)
  bool use_dsa = true;
  SolverParams solver;
};
void assemble_arrays(const ProblemArrays& in, HostProblem& out);
// pieces of assemble(), shared with assemble_arrays()
void build_stream_consts(HostProblem& hp);
void build_sip(HostProblem& hp);
void detect_uniform(HostProblem& hp);

// Boundary vector of one direction (operators.cpp:227-281).
void boundary_vector(const HostProblem& hp, const Field& g, int angle, double* out);

// proj/src/low_rank.cpp:15-37 (mt19937_64 + masked rejection bounded draws)
class SubsampleRng {
 public:
  explicit SubsampleRng(std::uint64_t seed) : engine_(seed) {}
  std::uint64_t draw_below(std::uint64_t n);
  std::vector<int> sample_without_replacement(std::vector<int> pool, int count);

 private:
  std::mt19937_64 engine_;
};

// proj/src/low_rank.cpp:254-266
int truncation_rank(const std::vector<double>& s, double eps_svd);

// Directions owned by `rank` of `nranks`: units are mirror pairs
// {(j1, j2), (j1, n_z-1-j2)} listed pair-index-major / azimuth-minor and dealt
// round-robin, so every rank spans all quadrants and pairs never split.
std::vector<int> partition_angles(int n_theta, int n_omega_z, int nranks, int rank);

// Low-rank sharding of a list of m work items (angles of one LR phase):
// rank k owns the contiguous block [k*bsz, min(m, (k+1)*bsz)), bsz =
// ceil(m / nranks), so an in-place all-gather of bsz-item segments restores
// the whole list in order on every rank.
struct ShardBlock {
  int begin = 0, end = 0, bsz = 0;
};
ShardBlock shard_block(int m, int nranks, int rank);

// Counter-based U[0,1) generator for the C5 per-(cell, direction) sources
// (SURVEY.md §8(d)); bit-identical on host and device.
inline double c5_uniform(std::uint64_t seed, std::uint64_t counter) {
  std::uint64_t z = counter * 0x9E3779B97F4A7C15ull + seed;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return static_cast<double>(z >> 11) * 0x1.0p-53;
}

}  // namespace cuda
}  // namespace rtlr
