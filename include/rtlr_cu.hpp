/*
 * rtlr_cu.hpp — header-only C++17 façade over the C ABI (rtlr_cu.h) with the
 * reference's own names and types (namespace rtlr::cuda), for a C++ caller
 * such as the reference tree itself.  Vectors are
 * std::vector<double> in the reference's DOF layout; matrices are
 * column-major (Matrix).  Errors surface as the reference's exception
 * classes: std::invalid_argument, std::runtime_error, rtlr::cuda::ConfigError.
 *
 * Reference interfaces mirrored (file:line under /root/reference/proj):
 *   sweep                        include/rtlr/sweep.hpp:14-15
 *   si_step, solve_full_rank     include/rtlr/full_rank.hpp:28-43
 *   DiffusionSystem solve/correct include/rtlr/diffusion.hpp:16-39
 *   SubsampleRng, LowRankParams, LowRankBasis, greedy_subsample,
 *   truncation_rank, truncate_factors, low_rank_si, solve_low_rank
 *                                include/rtlr/low_rank.hpp:18-158
 *   SolveReport, LowRankFactors  include/rtlr/report.hpp:12-44
 */
#ifndef RTLR_CU_HPP
#define RTLR_CU_HPP

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "rtlr_cu.h"

namespace rtlr {
namespace cuda {

using Vector = std::vector<double>;

struct Matrix {  // column-major rows x cols
  int rows = 0, cols = 0;
  std::vector<double> a;
  Matrix() = default;
  Matrix(int r, int c) : rows(r), cols(c), a(static_cast<size_t>(r) * c, 0.0) {}
  double& operator()(int i, int j) { return a[static_cast<size_t>(j) * rows + i]; }
  double operator()(int i, int j) const { return a[static_cast<size_t>(j) * rows + i]; }
  double* col(int j) { return a.data() + static_cast<size_t>(j) * rows; }
  const double* col(int j) const { return a.data() + static_cast<size_t>(j) * rows; }
};

struct ConfigError : std::runtime_error {  // problem.hpp:16-18
  using std::runtime_error::runtime_error;
};

inline void check(int rc) {
  if (rc == RTLR_CU_OK) return;
  const std::string m = rtlr_cu_last_error();
  if (rc == RTLR_CU_INVALID_ARGUMENT) throw std::invalid_argument(m);
  if (rc == RTLR_CU_CONFIG_ERROR) throw ConfigError(m);
  throw std::runtime_error(m);
}

struct FullRankOptions {  // full_rank.hpp:32-37
  double eps_si_sa = 1e-6;
  int max_iterations = 500;
  bool use_dsa = true;
  bool store_psi = true;
};
struct LowRankParams {  // low_rank.hpp:29-36
  int p = 1, q = 8;
  double eps_res = 1e-7, eps_diff = 1e-7, eps_svd = 1e-8, eps_mgs = 1e-10;
};
struct LowRankOptions {  // low_rank.hpp:146-153
  LowRankParams inner;
  double eps_si_sa = 1e-6;
  int max_iterations = 500;
  bool use_dsa = true;
  std::uint64_t seed = 0;
  bool build_factors = true;
};
struct OuterRecord {  // report.hpp:19-31
  double diff_two_norm = 0, diff_inf_norm = 0;
  int rank = -1;
  double oversampling = 0;
  int inner_iterations = 0, sampled_count = 0;
  bool fullrank_fallback = false;
};
struct LowRankFactors {  // report.hpp:12-17
  Matrix X, V;
  Vector S;
  int rank() const { return static_cast<int>(S.size()); }
};
struct SolveReport {  // report.hpp:33-44
  std::string method;
  Vector phi;
  bool converged = false;
  int iterations = 0;
  double solve_seconds = 0;
  long long psi_dofs = 0;
  std::vector<OuterRecord> history;
  bool has_psi = false;
  Matrix psi;
  bool has_factors = false;
  LowRankFactors factors;
  std::vector<std::vector<int>> sampled_log;
};

inline rtlr_cu_lr_params to_c(const LowRankParams& p) {
  rtlr_cu_lr_params c;
  c.p = p.p;
  c.q = p.q;
  c.eps_res = p.eps_res;
  c.eps_diff = p.eps_diff;
  c.eps_svd = p.eps_svd;
  c.eps_mgs = p.eps_mgs;
  return c;
}

// An assembled problem on one GPU: AssembledProblem (problem.hpp:98-106) from
// a preset / BASELINE config, or the caller's own operators (upload).
class Problem {
 public:
  Problem(const std::string& preset, int device) {
    rtlr_cu_config* cfg = nullptr;
    check(rtlr_cu_config_create(preset.c_str(), &cfg));
    const int rc = rtlr_cu_problem_create(cfg, device, &p_);
    rtlr_cu_config_destroy(cfg);
    check(rc);
    info();
  }
  explicit Problem(const rtlr_cu_problem_desc& d, int device) {
    check(rtlr_cu_problem_upload(&d, device, &p_));
    info();
  }
  Problem(const Problem&) = delete;
  Problem& operator=(const Problem&) = delete;
  ~Problem() { rtlr_cu_problem_destroy(p_); }
  rtlr_cu_problem* get() const { return p_; }
  int n_dofs() const { return static_cast<int>(info_[4]); }
  int n_omega() const { return static_cast<int>(info_[5]); }
  Vector host(const char* what, size_t n) const {
    Vector v(n);
    check(rtlr_cu_problem_get(p_, what, v.data()));
    return v;
  }

 private:
  void info() { check(rtlr_cu_problem_info(p_, info_)); }
  rtlr_cu_problem* p_ = nullptr;
  int64_t info_[8] = {};
};

// sweep(ops, quad, angle, rhs) (sweep.hpp:14-15)
inline Vector sweep(Problem& P, int angle, const Vector& rhs) {
  Vector psi(rhs.size());
  check(rtlr_cu_sweep(P.get(), &angle, 1, rhs.data(), 0, psi.data(), static_cast<int64_t>(rhs.size()), RTLR_CU_HOST));
  return psi;
}

// si_step (full_rank.hpp:28-30): phi_star
inline Vector si_step(Problem& P, const Vector& phi_prev) {
  Vector out(phi_prev.size());
  check(rtlr_cu_si_step(P.get(), phi_prev.data(), out.data(), nullptr, RTLR_CU_HOST));
  return out;
}

// DiffusionSystem::solve / correct (diffusion.hpp:16-39)
struct DiffusionSystem {
  Problem* P;
  explicit DiffusionSystem(Problem& p) : P(&p) {}
  Vector solve(const Vector& rhs) const {
    Vector x(rhs.size());
    check(rtlr_cu_dsa_solve(P->get(), rhs.data(), x.data(), RTLR_CU_HOST, nullptr));
    return x;
  }
  Vector correct(const Vector& phi_star, const Vector& phi_prev) const {
    Vector d(phi_star.size());
    check(rtlr_cu_dsa_correct(P->get(), phi_star.data(), phi_prev.data(), d.data(), RTLR_CU_HOST));
    return d;
  }
};

inline SolveReport report_of(rtlr_cu_report* r, const char* method, int n_omega) {
  int64_t info[8];
  check(rtlr_cu_report_info(r, info));
  SolveReport out;
  out.method = method;
  out.iterations = static_cast<int>(info[0]);
  out.converged = info[1] != 0;
  out.psi_dofs = info[6];
  out.phi.resize(static_cast<size_t>(info[7]));
  check(rtlr_cu_report_get(r, "phi", out.phi.data()));
  check(rtlr_cu_report_get(r, "solve_seconds", &out.solve_seconds));
  const int nh = static_cast<int>(info[2]);
  out.history.resize(nh);
  Vector col(nh > 0 ? nh : 1);
  auto column = [&](const char* name, auto set) {
    check(rtlr_cu_report_get(r, name, col.data()));
    for (int k = 0; k < nh; ++k) set(out.history[k], col[k]);
  };
  column("diff_two_norm", [](OuterRecord& o, double v) { o.diff_two_norm = v; });
  column("diff_inf_norm", [](OuterRecord& o, double v) { o.diff_inf_norm = v; });
  column("rank", [](OuterRecord& o, double v) { o.rank = static_cast<int>(v); });
  column("oversampling", [](OuterRecord& o, double v) { o.oversampling = v; });
  column("inner_iterations", [](OuterRecord& o, double v) { o.inner_iterations = static_cast<int>(v); });
  column("sampled_count", [](OuterRecord& o, double v) { o.sampled_count = static_cast<int>(v); });
  column("fullrank_fallback", [](OuterRecord& o, double v) { o.fullrank_fallback = v != 0; });
  std::vector<int> counts(nh > 0 ? nh : 1), flat(info[5] > 0 ? static_cast<size_t>(info[5]) : 1);
  check(rtlr_cu_report_sampled(r, counts.data(), flat.data()));
  size_t k = 0;
  for (int i = 0; i < nh; ++i) {
    out.sampled_log.emplace_back(flat.begin() + k, flat.begin() + k + counts[i]);
    k += counts[i];
  }
  const int fr = static_cast<int>(info[4]);
  if (fr > 0) {
    out.has_factors = true;
    out.factors.X = Matrix(static_cast<int>(out.phi.size()), fr);
    out.factors.V = Matrix(n_omega, fr);
    out.factors.S.resize(fr);
    check(rtlr_cu_report_get(r, "X", out.factors.X.a.data()));
    check(rtlr_cu_report_get(r, "V", out.factors.V.a.data()));
    check(rtlr_cu_report_get(r, "S", out.factors.S.data()));
  }
  if (info[3]) {
    out.has_psi = true;
    out.psi = Matrix(static_cast<int>(out.phi.size()), n_omega);
    check(rtlr_cu_report_get(r, "psi", out.psi.a.data()));
  }
  return out;
}

// solve_full_rank (full_rank.hpp:41-43)
inline SolveReport solve_full_rank(Problem& P, const FullRankOptions& o) {
  rtlr_cu_fr_options c;
  rtlr_cu_fr_options_default(&c);
  c.eps_si_sa = o.eps_si_sa;
  c.max_iterations = o.max_iterations;
  c.use_dsa = o.use_dsa;
  c.store_psi = o.store_psi;
  rtlr_cu_report* r = nullptr;
  check(rtlr_cu_solve_full_rank(P.get(), &c, &r));
  SolveReport out = report_of(r, "full", P.n_omega());
  rtlr_cu_report_destroy(r);
  return out;
}

// solve_low_rank (low_rank.hpp:156-158)
inline SolveReport solve_low_rank(Problem& P, const LowRankOptions& o) {
  rtlr_cu_lr_options c;
  rtlr_cu_lr_options_default(&c);
  c.p = o.inner.p;
  c.q = o.inner.q;
  c.eps_res = o.inner.eps_res;
  c.eps_diff = o.inner.eps_diff;
  c.eps_svd = o.inner.eps_svd;
  c.eps_mgs = o.inner.eps_mgs;
  c.eps_si_sa = o.eps_si_sa;
  c.max_iterations = o.max_iterations;
  c.use_dsa = o.use_dsa;
  c.seed = o.seed;
  c.build_factors = o.build_factors;
  rtlr_cu_report* r = nullptr;
  check(rtlr_cu_solve_low_rank(P.get(), &c, &r));
  SolveReport out = report_of(r, "lowrank", P.n_omega());
  rtlr_cu_report_destroy(r);
  return out;
}

// SubsampleRng (low_rank.hpp:18-27)
class SubsampleRng {
 public:
  explicit SubsampleRng(std::uint64_t seed) { check(rtlr_cu_rng_create(seed, &r_)); }
  SubsampleRng(const SubsampleRng&) = delete;
  SubsampleRng& operator=(const SubsampleRng&) = delete;
  ~SubsampleRng() { rtlr_cu_rng_destroy(r_); }
  std::uint64_t draw_below(std::uint64_t n) {
    std::uint64_t v = 0;
    check(rtlr_cu_rng_draw_below(r_, n, &v));
    return v;
  }
  std::vector<int> sample_without_replacement(std::vector<int> pool, int count) {
    std::vector<int> out(pool.size() + 1);
    int n = 0;
    check(rtlr_cu_rng_sample(r_, pool.data(), static_cast<int>(pool.size()), count, out.data(), &n));
    out.resize(n);
    return out;
  }
  rtlr_cu_rng* get() const { return r_; }

 private:
  rtlr_cu_rng* r_ = nullptr;
};

// LowRankBasis (low_rank.hpp:42-102)
class LowRankBasis {
 public:
  LowRankBasis(Problem& P, const Vector& rhs_core, const LowRankParams& prm = LowRankParams{}) : P_(&P) {
    const rtlr_cu_lr_params c = to_c(prm);
    check(rtlr_cu_lr_basis_create(P.get(), &c, rhs_core.data(), RTLR_CU_HOST, &b_));
  }
  LowRankBasis(const LowRankBasis&) = delete;
  LowRankBasis& operator=(const LowRankBasis&) = delete;
  ~LowRankBasis() { rtlr_cu_lr_basis_destroy(b_); }
  int rank() const { return static_cast<int>(info()[0]); }
  int snapshot_count() const { return static_cast<int>(info()[1]); }
  std::vector<int> sampled_angles() const {
    std::vector<int> s(snapshot_count() + 1);
    check(rtlr_cu_lr_basis_sampled(b_, s.data()));
    s.resize(snapshot_count());
    return s;
  }
  Matrix basis() const { return get("basis", P_->n_dofs(), rank()); }
  Matrix coefficient_record() const { return get("record", rank(), snapshot_count()); }
  Matrix projected_dx_minus() const { return get("dx_minus", rank(), rank()); }
  Matrix projected_dx_plus() const { return get("dx_plus", rank(), rank()); }
  Matrix projected_dy_minus() const { return get("dy_minus", rank(), rank()); }
  Matrix projected_dy_plus() const { return get("dy_plus", rank(), rank()); }
  Matrix projected_sigma_t() const { return get("sigma_t", rank(), rank()); }
  bool mgs_ro_update(const Matrix& snapshots, const std::vector<int>& angles, double eps_mgs,
                     double drop_tol = 1e-12) {
    int ro = 0;
    check(rtlr_cu_lr_mgs_ro_update(b_, snapshots.a.data(), angles.data(), static_cast<int>(angles.size()), eps_mgs,
                                   drop_tol, RTLR_CU_HOST, &ro));
    return ro != 0;
  }
  void update_projections(bool reorthogonalized) { check(rtlr_cu_lr_update_projections(b_, reorthogonalized)); }
  Vector galerkin_solve(int angle) const {
    Vector c(rank());
    check(rtlr_cu_lr_galerkin_solve(b_, &angle, 1, c.data(), RTLR_CU_HOST));
    return c;
  }
  double residual_norm(int angle, const Vector& c) const {
    double v = 0;
    check(rtlr_cu_lr_residual_norms(b_, &angle, 1, c.data(), &v, RTLR_CU_HOST));
    return v;
  }
  rtlr_cu_lr_basis* get() const { return b_; }

 private:
  std::vector<int64_t> info() const {
    std::vector<int64_t> i(4);
    check(rtlr_cu_lr_basis_info(b_, i.data()));
    return i;
  }
  Matrix get(const char* what, int rows, int cols) const {
    Matrix m(rows, cols);
    if (rows > 0 && cols > 0) check(rtlr_cu_lr_basis_get(b_, what, m.a.data(), RTLR_CU_HOST));
    return m;
  }
  Problem* P_;
  rtlr_cu_lr_basis* b_ = nullptr;
};

// SubsampleOutcome / greedy_subsample (low_rank.hpp:104-116)
struct SubsampleOutcome {
  std::vector<int> selected;
  double max_residual = 0.0;
  std::vector<int> candidates;
  std::vector<Vector> candidate_solutions;
  std::vector<double> residual_norms;
};
inline SubsampleOutcome greedy_subsample(const LowRankBasis& basis, const std::vector<char>& sampled_mask, int p,
                                         int q, SubsampleRng& rng) {
  const int r = basis.rank();
  std::vector<unsigned char> mask(sampled_mask.begin(), sampled_mask.end());
  std::vector<int> sel(p > 0 ? p : 1), cand(q > 0 ? q : 1);
  Vector sols(static_cast<size_t>(r) * (q > 0 ? q : 1)), norms(q > 0 ? q : 1);
  int ns = 0, nc = 0;
  SubsampleOutcome out;
  check(rtlr_cu_lr_greedy_subsample(basis.get(), mask.data(), p, q, rng.get(), sel.data(), &ns, &out.max_residual,
                                    cand.data(), &nc, sols.data(), norms.data(), RTLR_CU_HOST));
  out.selected.assign(sel.begin(), sel.begin() + ns);
  out.candidates.assign(cand.begin(), cand.begin() + nc);
  out.residual_norms.assign(norms.begin(), norms.begin() + nc);
  for (int k = 0; k < nc; ++k)
    out.candidate_solutions.emplace_back(sols.begin() + static_cast<size_t>(k) * r,
                                         sols.begin() + static_cast<size_t>(k + 1) * r);
  return out;
}

// truncation_rank / truncate_factors (low_rank.hpp:118-123)
inline int truncation_rank(const Vector& s, double eps_svd) {
  int r = 0;
  check(rtlr_cu_truncation_rank(s.data(), static_cast<int>(s.size()), eps_svd, &r));
  return r;
}
inline LowRankFactors truncate_factors(Problem& P, const Matrix& coefficients, const Matrix& basis, double eps_svd) {
  const int r = coefficients.rows;
  LowRankFactors f;
  Matrix X(basis.rows, r), V(coefficients.cols, r);
  Vector S(r);
  int k = 0;
  check(rtlr_cu_truncate_factors(P.get(), coefficients.a.data(), basis.a.data(), r, eps_svd, RTLR_CU_HOST, &k,
                                 X.a.data(), S.data(), V.a.data()));
  X.cols = V.cols = k;
  X.a.resize(static_cast<size_t>(X.rows) * k);
  V.a.resize(static_cast<size_t>(V.rows) * k);
  S.resize(k);
  f.X = std::move(X);
  f.V = std::move(V);
  f.S = std::move(S);
  return f;
}

// InnerLoopResult / low_rank_si (low_rank.hpp:125-144)
struct InnerLoopResult {
  Vector phi_star;
  Matrix coefficients, basis;
  int iterations = 0, rank = 0, sampled_count = 0, reorthogonalizations = 0, verification_rejections = 0;
  bool exhausted_all_angles = false;
  std::vector<int> sampled_order;
};
inline InnerLoopResult low_rank_si(Problem& P, const Vector& phi_prev, const LowRankParams& params,
                                   SubsampleRng& rng) {
  const rtlr_cu_lr_params c = to_c(params);
  rtlr_cu_inner* h = nullptr;
  check(rtlr_cu_low_rank_si(P.get(), phi_prev.data(), &c, rng.get(), RTLR_CU_HOST, &h));
  int64_t info[8];
  InnerLoopResult out;
  try {
    check(rtlr_cu_inner_info(h, info));
    out.iterations = static_cast<int>(info[0]);
    out.rank = static_cast<int>(info[1]);
    out.sampled_count = static_cast<int>(info[2]);
    out.reorthogonalizations = static_cast<int>(info[3]);
    out.verification_rejections = static_cast<int>(info[4]);
    out.exhausted_all_angles = info[5] != 0;
    const int n = static_cast<int>(info[6]), nom = static_cast<int>(info[7]);
    out.phi_star.resize(n);
    check(rtlr_cu_inner_get(h, "phi_star", out.phi_star.data(), RTLR_CU_HOST));
    out.coefficients = Matrix(out.rank, nom);
    out.basis = Matrix(n, out.rank);
    if (out.rank > 0) {
      check(rtlr_cu_inner_get(h, "coefficients", out.coefficients.a.data(), RTLR_CU_HOST));
      check(rtlr_cu_inner_get(h, "basis", out.basis.a.data(), RTLR_CU_HOST));
    }
    out.sampled_order.resize(out.sampled_count + 1);
    check(rtlr_cu_inner_sampled(h, out.sampled_order.data()));
    out.sampled_order.resize(out.sampled_count);
  } catch (...) {
    rtlr_cu_inner_destroy(h);
    throw;
  }
  rtlr_cu_inner_destroy(h);
  return out;
}

}  // namespace cuda
}  // namespace rtlr

#endif  // RTLR_CU_HPP
