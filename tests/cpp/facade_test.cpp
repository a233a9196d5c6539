// A C++ consumer of include/rtlr_cu.hpp, the rtlr::cuda façade a reference
// maintainer would include.  It compiles against the
// header alone and links librtlr_cu.so; with a GPU it drives the solvers
// and the low-rank primitives through the reference's names and checks the
// reference's own properties (test_low_rank.cpp, test_full_rank.cpp,
// test_diffusion.cpp).  `--no-gpu` runs the host-only entry points.
// Exit code 0 = every check passed.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>

#include "rtlr_cu.hpp"

using namespace rtlr::cuda;

static int failures = 0;
#define CHECK(cond)                                                   \
  do {                                                                \
    if (!(cond)) {                                                    \
      std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      ++failures;                                                     \
    }                                                                 \
  } while (0)

static double orth_error(const Matrix& x) {  // ||X^T X - I||_F
  double s = 0.0;
  for (int i = 0; i < x.cols; ++i)
    for (int j = 0; j < x.cols; ++j) {
      double d = 0.0;
      for (int k = 0; k < x.rows; ++k) d += x(k, i) * x(k, j);
      d -= (i == j) ? 1.0 : 0.0;
      s += d * d;
    }
  return std::sqrt(s);
}

static void host_checks() {
  CHECK(truncation_rank({1.0, 1e-4, 1e-12}, 1e-8) == 2);
  CHECK(truncation_rank({1.0, 1e-4, 1e-12}, 1e-2) == 1);
  CHECK(truncation_rank({0.0, 0.0, 0.0}, 1e-8) == 1);
  SubsampleRng a(1234), b(1234);
  std::vector<int> pool(128);
  for (int i = 0; i < 128; ++i) pool[i] = i;
  for (int t = 0; t < 20; ++t) CHECK(a.sample_without_replacement(pool, 3) == b.sample_without_replacement(pool, 3));
  bool threw = false;
  try {
    Problem p("no_such_preset", -1);
  } catch (const ConfigError&) {
    threw = true;
  }
  CHECK(threw);
}

static void gpu_checks() {
  // solve_full_rank on BASELINE C1: 12 outer iterations (the oracle's count)
  Problem c1("C1", 0);
  FullRankOptions fo;
  fo.eps_si_sa = 1e-8;
  fo.store_psi = false;
  SolveReport fr = solve_full_rank(c1, fo);
  CHECK(fr.converged && fr.iterations == 12);
  // DiffusionSystem::correct(phi, phi) == 0 exactly (test_diffusion.cpp:69)
  DiffusionSystem dsa(c1);
  Vector d = dsa.correct(fr.phi, fr.phi);
  double dmax = 0.0;
  for (double v : d) dmax = std::max(dmax, std::abs(v));
  CHECK(dmax == 0.0);

  // a caller-assembled problem: a preset's own arrays through upload
  Problem h("homogeneous(1,1)", -1);
  const int n = h.n_dofs(), nom = h.n_omega(), ncell = n / 4;
  Vector dirs = h.host("dirs", 3 * nom), w = h.host("weights", nom), st = h.host("sigma_t_blocks", 16 * ncell),
         ss = h.host("sigma_s_blocks", 16 * ncell), src = h.host("source", n);
  rtlr_cu_problem_desc desc;
  std::memset(&desc, 0, sizeof desc);
  desc.nx = desc.ny = 16;
  desc.x_min = desc.y_min = -1.0;
  desc.x_max = desc.y_max = 1.0;
  desc.n_theta = 8;
  desc.n_omega_z = 4;
  desc.n_omega = nom;
  desc.dirs = dirs.data();
  desc.weights = w.data();
  desc.sigma_t_blocks = st.data();
  desc.sigma_s_blocks = ss.data();
  desc.source = src.data();
  desc.use_dsa = 1;
  Problem u(desc, 0);
  Problem ref("homogeneous(1,1)", 0);
  LowRankOptions lo;
  lo.seed = 2024;
  SolveReport a = solve_low_rank(u, lo), b = solve_low_rank(ref, lo);
  CHECK(a.phi == b.phi && a.sampled_log == b.sampled_log && a.iterations == b.iterations);
  CHECK(a.has_factors && orth_error(a.factors.X) <= 1e-10 && orth_error(a.factors.V) <= 1e-10);

  // LowRankBasis: sweep snapshots, invariants (acceptance criterion 3 bars)
  Vector rhs_core = src;  // phi_prev = 0
  LowRankBasis basis(u, rhs_core);
  Matrix snaps(n, 3);
  for (int k = 0; k < 3; ++k) {
    Vector s = sweep(u, 5 * k, rhs_core);
    std::copy(s.begin(), s.end(), snaps.col(k));
  }
  const bool ro = basis.mgs_ro_update(snaps, {0, 5, 10}, 1e-10);
  basis.update_projections(ro);
  CHECK(basis.rank() == 3 && basis.snapshot_count() == 3);
  const Matrix x = basis.basis(), rec = basis.coefficient_record();
  CHECK(orth_error(x) <= 1e-10);
  double rerr = 0.0, rnorm = 0.0;
  for (int j = 0; j < 3; ++j)
    for (int i = 0; i < n; ++i) {
      double v = 0.0;
      for (int k = 0; k < 3; ++k) v += x(i, k) * rec(k, j);
      rerr += (v - snaps(i, j)) * (v - snaps(i, j));
      rnorm += snaps(i, j) * snaps(i, j);
    }
  CHECK(std::sqrt(rerr / rnorm) <= 1e-9);
  const Vector c = basis.galerkin_solve(5);  // reproduces its snapshot's record column
  double cerr = 0.0;
  for (int k = 0; k < 3; ++k) cerr = std::max(cerr, std::abs(c[k] - rec(k, 1)));
  CHECK(cerr <= 1e-8 * std::abs(rec(1, 1)));
  CHECK(basis.residual_norm(5, c) <= 1e-8);
  std::vector<char> mask(nom, 0);
  mask[0] = mask[5] = mask[10] = 1;
  SubsampleRng rng(42);
  SubsampleOutcome g = greedy_subsample(basis, mask, 2, 8, rng);
  CHECK(g.selected.size() == 2 && g.candidates.size() == 8);
  for (int s : g.selected) CHECK(!mask[s]);

  // low_rank_si against si_step (test_low_rank.cpp:390-412)
  SubsampleRng r2(7);
  LowRankParams prm;
  prm.q = 4;
  InnerLoopResult inner = low_rank_si(u, Vector(n, 0.0), prm, r2);
  Vector full = si_step(u, Vector(n, 0.0));
  double e = 0.0;
  for (int i = 0; i < n; ++i) e += (inner.phi_star[i] - full[i]) * (inner.phi_star[i] - full[i]);
  CHECK(std::sqrt(e) <= 1e-7);
  CHECK(inner.coefficients.rows == inner.rank && inner.coefficients.cols == nom);

  // reference errors: an out-of-range angle is invalid_argument
  bool threw = false;
  try {
    (void)basis.galerkin_solve(nom + 3);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  CHECK(threw);
}

int main(int argc, char** argv) {
  const bool gpu = !(argc > 1 && std::strcmp(argv[1], "--no-gpu") == 0);
  try {
    host_checks();
    if (gpu) gpu_checks();
  } catch (const std::exception& ex) {
    std::fprintf(stderr, "uncaught: %s\n", ex.what());
    return 1;
  }
  std::printf("facade_test: %s, %d failure(s)\n", gpu ? "gpu" : "host only", failures);
  return failures == 0 ? 0 : 1;
}
