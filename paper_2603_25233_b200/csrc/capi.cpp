// extern "C" layer (include/rtlr_cu.h) over rtlr::cuda.
#include <cuda_runtime.h>

#include <cstring>
#include <memory>
#include <string>

#include "../../include/rtlr_cu.h"
#include "capi_internal.hpp"
#include "dense.cuh"
#include "harness.hpp"
#include "problem.hpp"

using namespace rtlr::cuda;

namespace {

using namespace rtlr_capi;

void set_key(ProblemConfig& c, std::string k, double v) {
  for (const char* pre : {"mesh.", "quadrature.", "solver.", "domain.", "space."})
    if (k.rfind(pre, 0) == 0) k = k.substr(std::strlen(pre));
  SolverParams& s = c.solver;
  if (k == "nx") c.nx = static_cast<int>(v);
  else if (k == "ny") c.ny = static_cast<int>(v);
  else if (k == "n_theta") c.n_theta = static_cast<int>(v);
  else if (k == "n_omega_z") c.n_omega_z = static_cast<int>(v);
  else if (k == "degree") c.degree = static_cast<int>(v);
  else if (k == "x_min") c.x_min = v;
  else if (k == "x_max") c.x_max = v;
  else if (k == "y_min") c.y_min = v;
  else if (k == "y_max") c.y_max = v;
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
  else if (k == "sigma_s_const") c.sigma_s = [v](double, double) { return v; };
  else if (k == "sigma_a_const") c.sigma_a = [v](double, double) { return v; };
  else if (k == "source_const") c.source = [v](double, double) { return v; };
  else if (k == "boundary_const") {
    c.boundary = [v](double, double) { return v; };
    c.boundary_zero = (v == 0.0);
  } else
    throw ConfigError("config: unknown key '" + k + "'");
}

void put_vec(const std::vector<double>& v, double* out) { std::memcpy(out, v.data(), v.size() * sizeof(double)); }

}  // namespace

extern "C" {

const char* rtlr_cu_last_error(void) { return g_err.c_str(); }
int rtlr_cu_version(void) { return 1; }
int rtlr_cu_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

int rtlr_cu_config_create(const char* preset, rtlr_cu_config** out) {
  return guard([&] {
    need(preset && out, "config: null argument");
    auto c = std::make_unique<rtlr_cu_config>();
    c->cfg = make_config(preset);
    *out = c.release();
  });
}

int rtlr_cu_config_set(rtlr_cu_config* cfg, const char* key, double value) {
  return guard([&] {
    need(cfg && key, "config: null argument");
    set_key(cfg->cfg, key, value);
  });
}

int rtlr_cu_config_set_field(rtlr_cu_config* cfg, const char* which, rtlr_cu_field_fn fn, void* user) {
  return guard([&] {
    need(cfg && which && fn, "config: null argument");
    Field f = [fn, user](double x, double y) { return fn(user, x, y); };
    std::string w = which;
    if (w == "sigma_s") cfg->cfg.sigma_s = f;
    else if (w == "sigma_a") cfg->cfg.sigma_a = f;
    else if (w == "source") cfg->cfg.source = f;
    else if (w == "boundary") {
      cfg->cfg.boundary = f;
      cfg->cfg.boundary_zero = false;
    } else
      throw ConfigError("config: unknown field '" + w + "'");
  });
}

void rtlr_cu_config_destroy(rtlr_cu_config* cfg) { delete cfg; }

int rtlr_cu_config_parse(const char* text, rtlr_cu_config** out) {
  return guard([&] {
    need(text && out, "config: null argument");
    RunConfig rc = parse_config_text(text);
    auto c = std::make_unique<rtlr_cu_config>();
    c->cfg = std::move(rc.cfg);
    c->mode = rc.mode;
    *out = c.release();
  });
}

int rtlr_cu_config_load(const char* path, rtlr_cu_config** out) {
  return guard([&] {
    need(path && out, "config: null argument");
    RunConfig rc = load_config_file(path);
    auto c = std::make_unique<rtlr_cu_config>();
    c->cfg = std::move(rc.cfg);
    c->mode = rc.mode;
    *out = c.release();
  });
}

int rtlr_cu_config_set_mode(rtlr_cu_config* cfg, const char* mode) {
  return guard([&] {
    need(cfg && mode, "config: null argument");
    cfg->mode = run_mode_from_name(mode);
  });
}

int rtlr_cu_run(const rtlr_cu_config* cfg, int device, const int64_t* seeds, int nseeds, const char* out_dir,
                int log_flux, char* summary, size_t summary_cap, int* all_conv) {
  return guard([&] {
    need(cfg != nullptr && (nseeds == 0 || seeds != nullptr) && nseeds >= 0, "run: bad argument");
    validate_config(cfg->cfg);
    RunConfig rc{cfg->cfg, cfg->mode};
    std::vector<RunResult> results;
    std::string text;
    {
      Problem P(rc.cfg, device);  // assembled once for every seed (rtlr_bench batch)
      if (nseeds == 0) {
        results.push_back(run_assembled(rc, P));
        text += run_summary(results.back());
      } else {
        for (int i = 0; i < nseeds; ++i) {
          RunConfig c = rc;
          c.cfg.solver.seed = static_cast<std::uint64_t>(seeds[i]);
          results.push_back(run_assembled(c, P));
          text += run_summary(results.back());
        }
        text += batch_summary(results);
      }
    }
    if (out_dir && *out_dir) write_outputs(results, out_dir, log_flux != 0);
    bool ok = true;
    for (const RunResult& r : results) ok = ok && all_converged(r);
    if (all_conv) *all_conv = ok ? 1 : 0;
    if (summary && summary_cap > 0) {
      const size_t n = std::min(summary_cap - 1, text.size());
      std::memcpy(summary, text.data(), n);
      summary[n] = 0;
    }
  });
}

int rtlr_cu_problem_create(const rtlr_cu_config* cfg, int device, rtlr_cu_problem** out) {
  return guard([&] {
    need(cfg && out, "problem: null argument");
    auto p = std::make_unique<rtlr_cu_problem>();
    p->p = std::make_unique<Problem>(cfg->cfg, device);
    *out = p.release();
  });
}

void rtlr_cu_problem_destroy(rtlr_cu_problem* p) { delete p; }

int rtlr_cu_problem_fr_options(const rtlr_cu_problem* p, rtlr_cu_fr_options* o) {
  return guard([&] {
    need(p && o, "problem: null argument");
    const SolverParams& s = p->p->host().cfg.solver;  // report.cpp:20-27
    o->eps_si_sa = s.eps_si_sa;
    o->max_iterations = s.max_iterations;
    o->use_dsa = s.use_dsa;
    o->store_psi = s.store_psi;
  });
}

int rtlr_cu_problem_lr_options(const rtlr_cu_problem* p, rtlr_cu_lr_options* o) {
  return guard([&] {
    need(p && o, "problem: null argument");
    const SolverParams& s = p->p->host().cfg.solver;  // report.cpp:29-43
    o->p = s.p;
    o->q = s.q;
    o->eps_res = s.eps_res;
    o->eps_diff = s.eps_diff;
    o->eps_svd = s.eps_svd;
    o->eps_mgs = s.eps_mgs;
    o->eps_si_sa = s.eps_si_sa;
    o->max_iterations = s.max_iterations;
    o->use_dsa = s.use_dsa;
    o->seed = s.seed;
    o->build_factors = s.build_factors;
  });
}

int rtlr_cu_problem_info(const rtlr_cu_problem* p, int64_t info[8]) {
  return guard([&] {
    need(p && info, "problem: null argument");
    const HostProblem& h = p->p->host();
    info[0] = h.nx;
    info[1] = h.ny;
    info[2] = h.cfg.n_theta;
    info[3] = h.cfg.n_omega_z;
    info[4] = h.ndof;
    info[5] = h.n_omega;
    info[6] = static_cast<int64_t>(p->p->unique_rep().size());
    info[7] = h.sigma_t_uniform;
  });
}

int rtlr_cu_problem_degree(const rtlr_cu_problem* p, int* degree, int* dofs_per_cell) {
  return guard([&] {
    need(p && degree && dofs_per_cell, "problem: null argument");
    *degree = p->p->host().degree;
    *dofs_per_cell = p->p->host().spc;
  });
}

int rtlr_cu_problem_get(const rtlr_cu_problem* p, const char* what, double* out) {
  return guard([&] {
    need(p && what && out, "problem: null argument");
    const HostProblem& h = p->p->host();
    std::string w = what;
    if (w == "dirs") put_vec(h.dirs, out);
    else if (w == "weights") put_vec(h.weights, out);
    else if (w == "source") put_vec(h.source, out);
    else if (w == "sigma_t_blocks") put_vec(h.sigma_t, out);
    else if (w == "sigma_s_blocks") put_vec(h.sigma_s, out);
    else if (w == "sigma_a_blocks") put_vec(h.sigma_a, out);
    else if (w == "sip_bsr") put_vec(h.sip, out);
    else if (w == "stream_blocks" && h.degree != 1) put_vec(h.kblocks, out);
    else if (w == "stream_blocks") {
      const double* m[8] = {h.sc.ax_minus, h.sc.ax_plus, h.sc.ay_minus, h.sc.ay_plus,
                            h.sc.bx_minus, h.sc.bx_plus, h.sc.by_minus, h.sc.by_plus};
      for (int k = 0; k < 8; ++k) std::memcpy(out + 16 * k, m[k], 16 * sizeof(double));
    } else
      throw std::invalid_argument("problem_get: unknown field '" + w + "'");
  });
}

int rtlr_cu_problem_set_stream(rtlr_cu_problem* p, void* s) {
  return guard([&] {
    gpu(p).set_stream(static_cast<cudaStream_t>(s));
  });
}

int rtlr_cu_problem_set_option(rtlr_cu_problem* p, const char* key, double v) {
  return guard([&] {
    need(p && key, "problem: null argument");
    std::string k = key;
    if (k == "pcg_rtol") p->p->pcg_rtol = v;
    else if (k == "pcg_max_iters") p->p->pcg_max_iters = static_cast<int>(v);
    else if (k == "pcg_multigrid") p->p->pcg_multigrid = v != 0.0;
    else if (k == "profile_phases") p->p->profile_phases = v != 0.0;
    else if (k == "sweep_kernel") {
      need(v == 0.0 || v == 1.0 || v == 2.0 || v == 3.0 || v == 4.0 || v == 5.0 || v == 6.0,
           "sweep_kernel: 0 (auto), 1 (skewed wavefront), 2 (row scan), 3 (row scan, prefactored blocks), "
           "4 (cluster wavefront), 5 (direction groups, heterogeneous media, shared right-hand side), "
           "6 (general-degree diagonal wavefront)");
      p->p->sweep_kernel = static_cast<int>(v);
    } else throw std::invalid_argument("unknown option '" + k + "'");
  });
}

int rtlr_cu_synchronize(rtlr_cu_problem* p) {
  return guard([&] { RTLR_CUDA(cudaStreamSynchronize(gpu(p).stream())); });
}

int rtlr_cu_sweep(rtlr_cu_problem* p, const int* angles, int n, const double* rhs, int64_t rhs_stride,
                  double* psi, int64_t psi_stride, int where) {
  return guard([&] {
    need(p && rhs && psi && n >= 0, "sweep: null argument");
    Problem& P = gpu(p);
    const HostProblem& h = P.host();
    need(psi_stride >= h.ndof, "sweep: psi stride smaller than N_x");
    need(rhs_stride == 0 || rhs_stride >= h.ndof, "sweep: bad rhs stride");
    if (n == 0) return;
    std::vector<int> ang(n);
    for (int k = 0; k < n; ++k) {
      ang[k] = angles ? angles[k] : k;
      if (ang[k] < 0 || ang[k] >= h.n_omega) throw std::invalid_argument("sweep: angle index out of range");
    }
    if (where == RTLR_CU_HOST) {  // chunked, H2D / sweep / D2H overlapped
      P.sweep_host(ang.data(), n, rhs, rhs_stride, psi, psi_stride);
      return;
    }
    cudaStream_t s = P.stream();
    int* d_ang = nullptr;
    RTLR_CUDA(cudaMallocAsync(&d_ang, n * sizeof(int), s));
    RTLR_CUDA(cudaMemcpyAsync(d_ang, ang.data(), n * sizeof(int), cudaMemcpyHostToDevice, s));
    const size_t rhs_n = rhs_stride == 0 ? h.ndof : static_cast<size_t>(rhs_stride) * (n - 1) + h.ndof;
    In r(rhs, rhs_n, where, s);
    Out o(psi, static_cast<size_t>(psi_stride) * (n - 1) + h.ndof, where, s);
    // one shared right-hand side in a heterogeneous medium: direction groups
    if (!(rhs_stride == 0 && P.sweep_het(ang, nullptr, r.d, o.d, psi_stride, nullptr)))
      P.sweep(d_ang, n, r.d, rhs_stride, o.d, psi_stride);
    o.finish();
    cudaFreeAsync(d_ang, s);
    P.check_error();
  });
}

int rtlr_cu_sweep_async(rtlr_cu_problem* p, const int* d_angles, int n, const double* d_rhs,
                        int64_t rhs_stride, double* d_psi, int64_t psi_stride) {
  return guard([&] {
    Problem& P = gpu(p);
    need(d_rhs && d_psi && n >= 0, "sweep: null argument");
    need(psi_stride >= P.host().ndof, "sweep: psi stride smaller than N_x");
    need(rhs_stride == 0 || rhs_stride >= P.host().ndof, "sweep: bad rhs stride");
    P.sweep(d_angles, n, d_rhs, rhs_stride, d_psi, psi_stride);
  });
}

int rtlr_cu_check(rtlr_cu_problem* p) {
  return guard([&] { gpu(p).check_error(); });
}

int rtlr_cu_sweep_dirs(rtlr_cu_problem* p, const double* omega_xy, int n, const double* rhs,
                       int64_t rhs_stride, double* psi, int64_t psi_stride, int where) {
  return guard([&] {
    need(p && omega_xy && rhs && psi && n >= 0, "sweep: null argument");
    Problem& P = gpu(p);
    const HostProblem& h = P.host();
    need(psi_stride >= h.ndof, "sweep: psi stride smaller than N_x");
    if (n == 0) return;
    cudaStream_t s = P.stream();
    std::vector<double> d3(3 * static_cast<size_t>(n));
    for (int k = 0; k < n; ++k) {
      d3[3 * k] = omega_xy[2 * k];
      d3[3 * k + 1] = omega_xy[2 * k + 1];
      d3[3 * k + 2] = 0.0;
    }
    double* dd = nullptr;
    RTLR_CUDA(cudaMallocAsync(&dd, d3.size() * sizeof(double), s));
    RTLR_CUDA(cudaMemcpyAsync(dd, d3.data(), d3.size() * sizeof(double), cudaMemcpyHostToDevice, s));
    const size_t rhs_n = rhs_stride == 0 ? h.ndof : static_cast<size_t>(rhs_stride) * (n - 1) + h.ndof;
    In r(rhs, rhs_n, where, s);
    Out o(psi, static_cast<size_t>(psi_stride) * (n - 1) + h.ndof, where, s);
    P.sweep(nullptr, n, r.d, rhs_stride, o.d, psi_stride, false, dd);
    o.finish();
    cudaFreeAsync(dd, s);
    P.check_error();
  });
}

int rtlr_cu_apply(rtlr_cu_problem* p, double omx, double omy, const double* v, double* out, int where) {
  return guard([&] {
    need(p && v && out, "apply: null argument");
    Problem& P = gpu(p);
    const size_t n = P.host().ndof;
    In vin(v, n, where, P.stream());
    Out o(out, n, where, P.stream());
    P.apply(omx, omy, vin.d, o.d);
    o.finish();
  });
}

int rtlr_cu_rhs_core(rtlr_cu_problem* p, const double* phi, double* out, int where) {
  return guard([&] {
    need(p && phi && out, "rhs_core: null argument");
    Problem& P = gpu(p);
    const size_t n = P.host().ndof;
    In in(phi, n, where, P.stream());
    Out o(out, n, where, P.stream());
    P.rhs_core(in.d, o.d);
    o.finish();
  });
}

int rtlr_cu_si_step(rtlr_cu_problem* p, const double* phi_prev, double* phi_star, double* psi, int where) {
  return guard([&] {
    need(p && phi_prev && phi_star, "si_step: null argument");
    Problem& P = gpu(p);
    const size_t n = P.host().ndof;
    In in(phi_prev, n, where, P.stream());
    Out o(phi_star, n, where, P.stream());
    Out ps(psi, psi ? n * P.host().n_omega : 0, where, P.stream());
    P.si_step(in.d, o.d, ps.d);
    o.finish();
    ps.finish();
  });
}

int rtlr_cu_dsa_solve(rtlr_cu_problem* p, const double* rhs, double* x, int where, int* iterations) {
  return guard([&] {
    need(p && rhs && x, "dsa_solve: null argument");
    Problem& P = gpu(p);
    const size_t n = P.host().ndof;
    In in(rhs, n, where, P.stream());
    Out o(x, n, where, P.stream());
    const int it = P.dsa_solve(in.d, o.d);
    o.finish();
    if (iterations) *iterations = it;
  });
}

int rtlr_cu_dsa_correct(rtlr_cu_problem* p, const double* phi_star, const double* phi_prev, double* delta,
                        int where) {
  return guard([&] {
    need(p && phi_star && phi_prev && delta, "dsa_correct: null argument");
    Problem& P = gpu(p);
    const size_t n = P.host().ndof;
    In a(phi_star, n, where, P.stream());
    In b(phi_prev, n, where, P.stream());
    Out o(delta, n, where, P.stream());
    P.dsa_correct(a.d, b.d, o.d);
    o.finish();
  });
}

int rtlr_cu_c5_fill(rtlr_cu_problem* p, double* d_rhs, int64_t n_dirs, int64_t dir0, uint64_t seed) {
  return guard([&] {
    need(p && d_rhs, "c5_fill: null argument");
    launch_c5_fill(d_rhs, n_dirs, dir0, gpu(p).host().ndof, seed, p->p->stream());
  });
}

void rtlr_cu_fr_options_default(rtlr_cu_fr_options* o) {
  FullRankOptions d;
  o->eps_si_sa = d.eps_si_sa;
  o->max_iterations = d.max_iterations;
  o->use_dsa = d.use_dsa;
  o->store_psi = d.store_psi;
}

void rtlr_cu_lr_options_default(rtlr_cu_lr_options* o) {
  LowRankOptions d;
  o->p = d.inner.p;
  o->q = d.inner.q;
  o->eps_res = d.inner.eps_res;
  o->eps_diff = d.inner.eps_diff;
  o->eps_svd = d.inner.eps_svd;
  o->eps_mgs = d.inner.eps_mgs;
  o->eps_si_sa = d.eps_si_sa;
  o->max_iterations = d.max_iterations;
  o->use_dsa = d.use_dsa;
  o->seed = d.seed;
  o->build_factors = d.build_factors;
}

int rtlr_cu_solve_full_rank(rtlr_cu_problem* p, const rtlr_cu_fr_options* o, rtlr_cu_report** out) {
  return guard([&] {
    need(p && o && out, "solve_full_rank: null argument");
    FullRankOptions fo;
    fo.eps_si_sa = o->eps_si_sa;
    fo.max_iterations = o->max_iterations;
    fo.use_dsa = o->use_dsa != 0;
    fo.store_psi = o->store_psi != 0;
    auto r = std::make_unique<rtlr_cu_report>();
    r->r = gpu(p).solve_full_rank(fo);
    *out = r.release();
  });
}

int rtlr_cu_solve_low_rank(rtlr_cu_problem* p, const rtlr_cu_lr_options* o, rtlr_cu_report** out) {
  return guard([&] {
    need(p && o && out, "solve_low_rank: null argument");
    LowRankOptions lo;
    lo.inner.p = o->p;
    lo.inner.q = o->q;
    lo.inner.eps_res = o->eps_res;
    lo.inner.eps_diff = o->eps_diff;
    lo.inner.eps_svd = o->eps_svd;
    lo.inner.eps_mgs = o->eps_mgs;
    lo.eps_si_sa = o->eps_si_sa;
    lo.max_iterations = o->max_iterations;
    lo.use_dsa = o->use_dsa != 0;
    lo.seed = o->seed;
    lo.build_factors = o->build_factors != 0;
    auto r = std::make_unique<rtlr_cu_report>();
    r->r = gpu(p).solve_low_rank(lo);
    *out = r.release();
  });
}

int rtlr_cu_report_info(const rtlr_cu_report* r, int64_t info[8]) {
  return guard([&] {
    need(r && info, "report: null argument");
    const SolveReport& s = r->r;
    info[0] = s.iterations;
    info[1] = s.converged;
    info[2] = static_cast<int64_t>(s.history.size());
    info[3] = s.has_psi;
    info[4] = s.has_factors ? s.factors.rank : -1;
    int64_t tot = 0;
    for (auto& v : s.sampled_log) tot += static_cast<int64_t>(v.size());
    info[5] = tot;
    info[6] = s.psi_dofs;
    info[7] = static_cast<int64_t>(s.phi.size());
  });
}

int rtlr_cu_report_get(const rtlr_cu_report* r, const char* what, double* out) {
  return guard([&] {
    need(r && what && out, "report: null argument");
    const SolveReport& s = r->r;
    std::string w = what;
    if (w == "phi") put_vec(s.phi, out);
    else if (w == "psi") put_vec(s.psi, out);
    else if (w == "S") put_vec(s.factors.S, out);
    else if (w == "X") put_vec(s.factors.X, out);
    else if (w == "V") put_vec(s.factors.V, out);
    else if (w == "solve_seconds") out[0] = s.solve_seconds;
    else if (w == "phase_work") {
      need(!s.phase_work.empty(), "report_get: phase_work is a low-rank report field");
      put_vec(s.phase_work, out);
    }
    else
      for (size_t i = 0; i < s.history.size(); ++i) {
        const OuterRecord& h = s.history[i];
        if (w == "diff_two_norm") out[i] = h.diff_two_norm;
        else if (w == "diff_inf_norm") out[i] = h.diff_inf_norm;
        else if (w == "rank") out[i] = h.rank;
        else if (w == "oversampling") out[i] = h.oversampling;
        else if (w == "inner_iterations") out[i] = h.inner_iterations;
        else if (w == "sampled_count") out[i] = h.sampled_count;
        else if (w == "fullrank_fallback") out[i] = h.fullrank_fallback;
        else if (w == "dsa_iterations") out[i] = h.dsa_iterations;
        else throw std::invalid_argument("report_get: unknown field '" + w + "'");
      }
  });
}

int rtlr_cu_report_sampled(const rtlr_cu_report* r, int* counts, int* flat) {
  return guard([&] {
    need(r && counts && flat, "report: null argument");
    size_t k = 0;
    for (size_t i = 0; i < r->r.sampled_log.size(); ++i) {
      counts[i] = static_cast<int>(r->r.sampled_log[i].size());
      for (int v : r->r.sampled_log[i]) flat[k++] = v;
    }
  });
}

void rtlr_cu_report_destroy(rtlr_cu_report* r) { delete r; }

int rtlr_cu_partition_angles(int n_theta, int n_omega_z, int nranks, int rank, int* count, int* angles) {
  return guard([&] {
    need(count != nullptr, "partition_angles: bad argument");
    const std::vector<int> a = partition_angles(n_theta, n_omega_z, nranks, rank);
    *count = static_cast<int>(a.size());
    if (angles) std::memcpy(angles, a.data(), a.size() * sizeof(int));
  });
}

int rtlr_cu_psi_difference(rtlr_cu_problem* p, const double* psi_full, const double* X, const double* S,
                           const double* V, int rank, double* out, int where) {
  return guard([&] {
    need(p && psi_full && out && rank >= 0 && (rank == 0 || (X && S && V)), "psi_difference: bad argument");
    Problem& P = gpu(p);
    const size_t n = P.host().ndof, nom = P.host().n_omega;
    In ps(psi_full, n * nom, where, P.stream()), x(X, n * rank, where, P.stream()), sv(S, rank, where, P.stream()),
        v(V, nom * rank, where, P.stream());
    *out = P.psi_difference(ps.d, x.d, sv.d, v.d, rank);
  });
}

int rtlr_cu_dense_qr(int device, int64_t m, int n, const double* a, double* q, double* r) {
  return guard([&] {
    need(m >= n && n >= 1 && a && q && r, "dense_qr: need m >= n >= 1 and host buffers");
    RTLR_CUDA(cudaSetDevice(device));
    cudaStream_t s;
    RTLR_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    const size_t mn = static_cast<size_t>(m) * n;
    DBuf<double> da, dq, dr, dt, dw;
    da.upload(a, mn, s);
    const size_t nw = householder_qr_work(m, n);
    householder_qr(m, n, da.get(), m, dt.ensure(n), dq.ensure(mn), m, dr.ensure(static_cast<size_t>(n) * n),
                   dw.ensure(nw), nw, s);
    RTLR_CUDA(cudaMemcpyAsync(q, dq.get(), mn * sizeof(double), cudaMemcpyDeviceToHost, s));
    RTLR_CUDA(cudaMemcpyAsync(r, dr.get(), static_cast<size_t>(n) * n * sizeof(double), cudaMemcpyDeviceToHost, s));
    RTLR_CUDA(cudaStreamSynchronize(s));
    RTLR_CUDA(cudaStreamDestroy(s));
  });
}

int rtlr_cu_dense_galerkin_border(int device, int r0, int k, int m, const int* angles, int n_omega,
                                  const double* dirs, const double* proj, const double* prhs, double* sol_full,
                                  double* sol_border) {
  return guard([&] {
    need(r0 >= 1 && k >= 0 && m >= 1 && m <= 64 && angles && dirs && proj && prhs && sol_full && sol_border,
         "dense_galerkin_border: bad argument");
    need(galerkin_border_fits(r0, k), "dense_galerkin_border: rank or border out of range");
    RTLR_CUDA(cudaSetDevice(device));
    cudaStream_t s;
    RTLR_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    const int r = r0 + k;
    const size_t rr = static_cast<size_t>(r) * r;
    DBuf<double> dd, dp, dr, w1, w2, s1, s2;
    DBuf<int> da, fl;
    dd.upload(dirs, 3 * static_cast<size_t>(n_omega), s);
    dp.upload(proj, 5 * rr, s);
    dr.upload(prhs, r, s);
    da.upload(angles, m, s);
    fl.ensure(2 * m);
    s1.ensure(static_cast<size_t>(r) * m);
    s2.ensure(static_cast<size_t>(r) * m);
    const size_t lw = galerkin_work_doubles(r, m);
    galerkin_batch(r, m, da.get(), dd.get(), dp.get(), r, rr, dr.get(), nullptr, s1.get(), r, fl.get(),
                   lw ? w1.ensure(lw) : nullptr, s);
    double* pw = w2.ensure(static_cast<size_t>(m) * galerkin_work_per_system(r0));
    galerkin_prefactor(r0, m, da.get(), dd.get(), dp.get(), r, rr, dr.get(), pw, s);
    galerkin_border_solve(r0, k, m, da.get(), dd.get(), dp.get(), r, rr, dr.get(), pw, s2.get(), r, fl.get() + m, s);
    RTLR_CUDA(cudaMemcpyAsync(sol_full, s1.get(), static_cast<size_t>(r) * m * sizeof(double), cudaMemcpyDeviceToHost, s));
    RTLR_CUDA(cudaMemcpyAsync(sol_border, s2.get(), static_cast<size_t>(r) * m * sizeof(double), cudaMemcpyDeviceToHost, s));
    RTLR_CUDA(cudaStreamSynchronize(s));
    RTLR_CUDA(cudaStreamDestroy(s));
  });
}

int rtlr_cu_shard_block(int m, int nranks, int rank, int* begin, int* end, int* bsz) {
  return guard([&] {
    need(begin != nullptr && end != nullptr && bsz != nullptr, "shard_block: null argument");
    const ShardBlock b = shard_block(m, nranks, rank);
    *begin = b.begin;
    *end = b.end;
    *bsz = b.bsz;
  });
}

int rtlr_cu_nccl_unique_id(unsigned char* out) {
  return guard([&] {
    need(out != nullptr, "nccl_unique_id: null argument");
    nccl_unique_id(out);
  });
}

int rtlr_cu_problem_set_comm(rtlr_cu_problem* p, int nranks, int rank, const unsigned char* id) {
  return guard([&] { gpu(p).set_comm(nranks, rank, id); });
}

}  // extern "C"
