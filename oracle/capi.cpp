// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp header).
// extern "C" surface so tests/ (ctypes) can drive the CPU restatement.
#include <cstring>
#include <memory>
#include <string>

#include "oracle.hpp"

using namespace oracle;

namespace {
thread_local std::string g_err;

struct Problem {
  ProblemSpec spec;
  std::unique_ptr<AssembledProblem> asm_;
};

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = std::string("invalid_argument: ") + e.what();
    return -1;
  } catch (const std::exception& e) {
    g_err = std::string("runtime_error: ") + e.what();
    return -2;
  }
}

void put(const Vec& v, double* out) { std::memcpy(out, v.data(), v.size() * sizeof(double)); }

void put_blocks(const std::vector<Mat>& b, double* out) {
  size_t k = 0;
  for (const Mat& m : b)
    for (double v : m.a) out[k++] = v;
}

std::vector<Mat> diag_blocks(const Csr& a, int s) {
  std::vector<Mat> out(a.n / s, Mat(s, s));
  for (int i = 0; i < a.n; ++i)
    for (int k = a.rowptr[i]; k < a.rowptr[i + 1]; ++k) {
      int j = a.colidx[k];
      if (j / s == i / s) out[i / s](i % s, j % s) = a.val[k];
    }
  return out;
}

const Csr& pick_csr(Problem* p, const std::string& w) {
  const DiscreteOperators& o = p->asm_->ops;
  if (w == "d_x_minus") return o.d_x_minus;
  if (w == "d_x_plus") return o.d_x_plus;
  if (w == "d_y_minus") return o.d_y_minus;
  if (w == "d_y_plus") return o.d_y_plus;
  if (w == "sigma_s") return o.sigma_s;
  if (w == "sigma_t") return o.sigma_t;
  if (w == "sigma_a") return o.sigma_a;
  if (w == "sip") return p->asm_->dsa->matrix();
  throw std::invalid_argument("unknown matrix " + w);
}
}  // namespace

extern "C" {

const char* oracle_last_error() { return g_err.c_str(); }

int oracle_gauss_legendre(int n, double* nodes, double* w) {
  return guard([&] {
    GaussLegendre g = gauss_legendre(n);
    put(g.nodes, nodes);
    put(g.weights, w);
  });
}

int oracle_quadrature(int nt, int nz, double* dirs, double* w) {
  return guard([&] {
    AngularQuadrature q = build_cl_quadrature(nt, nz);
    put(q.dirs, dirs);
    put(q.weights, w);
  });
}

double oracle_c5_uniform(unsigned long long seed, unsigned long long counter) {
  return c5_uniform(seed, counter);
}

void oracle_c5_fill(unsigned long long seed, long long dir0, long long ndirs, long long ndof, double* out) {
  for (long long k = 0; k < ndirs; ++k)
    for (long long i = 0; i < ndof; ++i)
      out[k * ndof + i] = c5_uniform(seed, static_cast<unsigned long long>((dir0 + k) * ndof + i));
}

int oracle_truncation_rank(const double* s, int n, double eps) {
  return truncation_rank(Vec(s, s + n), eps);
}

int oracle_svd_values(const double* a, int m, int n, double* s) {
  return guard([&] {
    Mat x(m, n);
    std::memcpy(x.a.data(), a, sizeof(double) * m * n);
    put(svd_values(x), s);
  });
}

void* oracle_problem_new(const char* name) {
  Problem* p = nullptr;
  int rc = guard([&] {
    p = new Problem;
    p->spec = make_problem(name);
  });
  if (rc != 0) {
    delete p;
    return nullptr;
  }
  return p;
}

void oracle_problem_free(void* h) { delete static_cast<Problem*>(h); }

int oracle_problem_set(void* h, const char* key, double v) {
  return guard([&] {
    ProblemSpec& s = static_cast<Problem*>(h)->spec;
    std::string k = key;
    if (k == "nx") s.nx = static_cast<int>(v);
    else if (k == "ny") s.ny = static_cast<int>(v);
    else if (k == "n_theta") s.n_theta = static_cast<int>(v);
    else if (k == "n_omega_z") s.n_omega_z = static_cast<int>(v);
    else if (k == "degree") s.degree = static_cast<int>(v);
    else if (k == "x_min") s.x_min = v;
    else if (k == "x_max") s.x_max = v;
    else if (k == "y_min") s.y_min = v;
    else if (k == "y_max") s.y_max = v;
    else if (k == "eps_si_sa") s.eps_si_sa = v;
    else if (k == "eps_res") s.eps_res = v;
    else if (k == "eps_diff") s.eps_diff = v;
    else if (k == "eps_svd") s.eps_svd = v;
    else if (k == "eps_mgs") s.eps_mgs = v;
    else if (k == "p") s.p = static_cast<int>(v);
    else if (k == "q") s.q = static_cast<int>(v);
    else if (k == "seed") s.seed = static_cast<std::uint64_t>(v);
    else if (k == "max_iterations") s.max_iterations = static_cast<int>(v);
    else if (k == "use_dsa") s.use_dsa = v != 0.0;
    else if (k == "store_psi") s.store_psi = v != 0.0;
    else if (k == "build_factors") s.build_factors = v != 0.0;
    else if (k == "dsa_factor") s.dsa_factor = v != 0.0;
    else if (k == "sigma_s_const") s.sigma_s = [v](double, double) { return v; };
    else if (k == "sigma_a_const") s.sigma_a = [v](double, double) { return v; };
    else if (k == "source_const") s.source = [v](double, double) { return v; };
    else if (k == "boundary_const") {
      s.boundary = [v](double, double) { return v; };
      s.boundary_zero = (v == 0.0);
    } else
      throw std::invalid_argument("unknown key " + k);
  });
}

// A ScalarField (dg_space.hpp:10) as a C callback, for "sigma_s" | "sigma_a"
// | "source" | "boundary" (the same callable the product's
// rtlr_cu_config_set_field takes).
int oracle_problem_set_field(void* h, const char* which, double (*fn)(void*, double, double), void* user) {
  return guard([&] {
    ProblemSpec& s = static_cast<Problem*>(h)->spec;
    if (!fn) throw std::invalid_argument("null field");
    Field f = [fn, user](double x, double y) { return fn(user, x, y); };
    std::string w = which;
    if (w == "sigma_s") s.sigma_s = f;
    else if (w == "sigma_a") s.sigma_a = f;
    else if (w == "source") s.source = f;
    else if (w == "boundary") {
      s.boundary = f;
      s.boundary_zero = false;
    } else
      throw std::invalid_argument("unknown field " + w);
  });
}

int oracle_problem_assemble(void* h) {
  return guard([&] {
    Problem* p = static_cast<Problem*>(h);
    p->asm_ = std::make_unique<AssembledProblem>();
    assemble_problem(p->spec, *p->asm_);
  });
}

// out: nx, ny, n_theta, n_omega_z, n_dofs, n_omega, degree, bc_any
int oracle_problem_info(void* h, long long* out) {
  return guard([&] {
    Problem* p = static_cast<Problem*>(h);
    const ProblemSpec& s = p->spec;
    out[0] = s.nx;
    out[1] = s.ny;
    out[2] = s.n_theta;
    out[3] = s.n_omega_z;
    out[4] = p->asm_ ? p->asm_->space.size() : 0;
    out[5] = static_cast<long long>(s.n_theta) * s.n_omega_z;
    out[6] = s.degree;
    out[7] = p->asm_ ? p->asm_->bc.any : 0;
  });
}

int oracle_problem_get(void* h, const char* what, double* out) {
  return guard([&] {
    Problem* p = static_cast<Problem*>(h);
    AssembledProblem& a = *p->asm_;
    std::string w = what;
    const int s = a.space.dofs_per_cell();
    if (w == "source") put(a.source, out);
    else if (w == "dirs") put(a.quad.dirs, out);
    else if (w == "weights") put(a.quad.weights, out);
    else if (w == "sigma_t_blocks") put_blocks(a.ops.sigma_t_blocks, out);
    else if (w == "sigma_s_blocks") put_blocks(diag_blocks(a.ops.sigma_s, s), out);
    else if (w == "sigma_a_blocks") put_blocks(diag_blocks(a.ops.sigma_a, s), out);
    else if (w == "stream_blocks") {  // ax-,ax+,ay-,ay+,bx-,bx+,by-,by+ (each s*s col-major)
      const Mat* m[8] = {&a.ops.ax_minus, &a.ops.ax_plus, &a.ops.ay_minus, &a.ops.ay_plus,
                         &a.ops.bx_minus, &a.ops.bx_plus, &a.ops.by_minus, &a.ops.by_plus};
      size_t k = 0;
      for (const Mat* mm : m)
        for (double v : mm->a) out[k++] = v;
    } else
      throw std::invalid_argument("unknown field " + w);
  });
}

long long oracle_problem_nnz(void* h, const char* which) {
  long long nnz = -1;
  guard([&] { nnz = static_cast<long long>(pick_csr(static_cast<Problem*>(h), which).val.size()); });
  return nnz;
}

int oracle_problem_csr(void* h, const char* which, int* rowptr, int* colidx, double* val) {
  return guard([&] {
    const std::string w(which);
    const Csr& m = pick_csr(static_cast<Problem*>(h), w);
    std::memcpy(rowptr, m.rowptr.data(), sizeof(int) * m.rowptr.size());
    std::memcpy(colidx, m.colidx.data(), sizeof(int) * m.colidx.size());
    std::memcpy(val, m.val.data(), sizeof(double) * m.val.size());
  });
}

int oracle_sweep(void* h, double omx, double omy, const double* rhs, double* psi) {
  return guard([&] {
    AssembledProblem& a = *static_cast<Problem*>(h)->asm_;
    Vec r(rhs, rhs + a.space.size());
    put(sweep(a.ops, omx, omy, r), psi);
  });
}

int oracle_apply(void* h, double omx, double omy, const double* v, double* out) {
  return guard([&] {
    AssembledProblem& a = *static_cast<Problem*>(h)->asm_;
    Vec x(v, v + a.space.size());
    put(upwind_combination(a.ops, omx, omy).apply(x), out);
  });
}

int oracle_rhs_core(void* h, const double* phi, double* out) {
  return guard([&] {
    AssembledProblem& a = *static_cast<Problem*>(h)->asm_;
    Vec x(phi, phi + a.space.size());
    Vec r = a.ops.sigma_s.mul(x);
    for (size_t i = 0; i < r.size(); ++i) r[i] += a.source[i];
    put(r, out);
  });
}

int oracle_boundary_vector(void* h, int angle, double* out) {
  return guard([&] {
    Problem* p = static_cast<Problem*>(h);
    AssembledProblem& a = *p->asm_;
    if (!p->spec.boundary) throw std::invalid_argument("no boundary field");
    put(boundary_vector(a.space, a.quad, p->spec.boundary, angle), out);
  });
}

int oracle_boundary_vector_dir(void* h, double omx, double omy, double* out) {
  return guard([&] {
    Problem* p = static_cast<Problem*>(h);
    AssembledProblem& a = *p->asm_;
    if (!p->spec.boundary) throw std::invalid_argument("no boundary field");
    AngularQuadrature q;
    q.n_theta = q.n_omega_z = 1;
    q.dirs = {omx, omy, 0.0};
    q.weights = {1.0};
    put(boundary_vector(a.space, q, p->spec.boundary, 0), out);
  });
}

int oracle_dsa_solve(void* h, const double* rhs, double* out) {
  return guard([&] {
    AssembledProblem& a = *static_cast<Problem*>(h)->asm_;
    if (!a.dsa) throw std::invalid_argument("no diffusion system");
    put(a.dsa->solve(Vec(rhs, rhs + a.space.size())), out);
  });
}

int oracle_dsa_correct(void* h, const double* phi_star, const double* phi_prev, double* out) {
  return guard([&] {
    AssembledProblem& a = *static_cast<Problem*>(h)->asm_;
    const int n = a.space.size();
    put(a.dsa->correct(Vec(phi_star, phi_star + n), Vec(phi_prev, phi_prev + n)), out);
  });
}

int oracle_si_step(void* h, const double* phi_prev, double* phi_star, double* psi_or_null) {
  return guard([&] {
    AssembledProblem& a = *static_cast<Problem*>(h)->asm_;
    const int n = a.space.size();
    SIStepResult r = si_step(a.ops, a.quad, a.bc, a.source, Vec(phi_prev, phi_prev + n));
    put(r.phi_star, phi_star);
    if (psi_or_null) put(r.psi.a, psi_or_null);
  });
}

void* oracle_solve(void* h, const char* method) {
  SolveReport* rep = nullptr;
  int rc = guard([&] {
    Problem* p = static_cast<Problem*>(h);
    AssembledProblem& a = *p->asm_;
    const ProblemSpec& s = p->spec;
    std::string m = method;
    if (m == "full") {
      FullRankOptions o;
      o.eps_si_sa = s.eps_si_sa;
      o.max_iterations = s.max_iterations;
      o.use_dsa = s.use_dsa;
      o.store_psi = s.store_psi;
      rep = new SolveReport(solve_full_rank(a.ops, a.quad, a.bc, a.source, a.dsa, o));
    } else if (m == "lowrank") {
      LowRankOptions o;
      o.inner.p = s.p;
      o.inner.q = s.q;
      o.inner.eps_res = s.eps_res;
      o.inner.eps_diff = s.eps_diff;
      o.inner.eps_svd = s.eps_svd;
      o.inner.eps_mgs = s.eps_mgs;
      o.eps_si_sa = s.eps_si_sa;
      o.max_iterations = s.max_iterations;
      o.use_dsa = s.use_dsa;
      o.seed = s.seed;
      o.build_factors = s.build_factors;
      rep = new SolveReport(solve_low_rank(a.ops, a.quad, a.bc, a.source, a.dsa, o));
    } else {
      throw std::invalid_argument("unknown method " + m);
    }
  });
  return rc == 0 ? rep : nullptr;
}

void oracle_result_free(void* r) { delete static_cast<SolveReport*>(r); }

// out: iterations, converged, n_history, has_psi, factor_rank, sampled_total, psi_dofs
int oracle_result_info(void* r, long long* out) {
  return guard([&] {
    SolveReport* s = static_cast<SolveReport*>(r);
    out[0] = s->iterations;
    out[1] = s->converged;
    out[2] = static_cast<long long>(s->history.size());
    out[3] = s->has_psi;
    out[4] = s->has_factors ? s->factors.rank() : -1;
    long long tot = 0;
    for (auto& v : s->sampled_log) tot += static_cast<long long>(v.size());
    out[5] = tot;
    out[6] = s->psi_dofs;
  });
}

int oracle_result_get(void* r, const char* what, double* out) {
  return guard([&] {
    SolveReport* s = static_cast<SolveReport*>(r);
    std::string w = what;
    if (w == "phi") put(s->phi, out);
    else if (w == "solve_seconds") out[0] = s->solve_seconds;
    else if (w == "psi") put(s->psi.a, out);
    else if (w == "S") put(s->factors.S, out);
    else if (w == "X") put(s->factors.X.a, out);
    else if (w == "V") put(s->factors.V.a, out);
    else {
      for (size_t i = 0; i < s->history.size(); ++i) {
        const OuterRecord& h = s->history[i];
        if (w == "diff_two_norm") out[i] = h.diff_two_norm;
        else if (w == "diff_inf_norm") out[i] = h.diff_inf_norm;
        else if (w == "rank") out[i] = h.rank;
        else if (w == "oversampling") out[i] = h.oversampling;
        else if (w == "inner_iterations") out[i] = h.inner_iterations;
        else if (w == "sampled_count") out[i] = h.sampled_count;
        else if (w == "fullrank_fallback") out[i] = h.fullrank_fallback;
        else throw std::invalid_argument("unknown result field " + w);
      }
    }
  });
}

int oracle_result_sampled(void* r, int* counts, int* flat) {
  return guard([&] {
    SolveReport* s = static_cast<SolveReport*>(r);
    size_t k = 0;
    for (size_t i = 0; i < s->sampled_log.size(); ++i) {
      counts[i] = static_cast<int>(s->sampled_log[i].size());
      for (int v : s->sampled_log[i]) flat[k++] = v;
    }
  });
}

double oracle_psi_difference(void* full, void* low) {
  double d = -1.0;
  guard([&] {
    d = psi_difference(static_cast<SolveReport*>(full)->psi, static_cast<SolveReport*>(low)->factors);
  });
  return d;
}

}  // extern "C"
