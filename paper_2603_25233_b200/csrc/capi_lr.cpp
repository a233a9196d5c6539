// extern "C" layer, part 2: caller-assembled problems and the reference's
// low-rank primitives (include/rtlr_cu.h, "caller-assembled problems" and
// "low-rank primitives"), over rtlr::cuda::LowRankEngine.
#include <cuda_runtime.h>

#include <algorithm>
#include <memory>
#include <vector>

#include "../../include/rtlr_cu.h"
#include "capi_internal.hpp"
#include "lowrank.hpp"

using namespace rtlr::cuda;
using namespace rtlr_capi;

struct rtlr_cu_rng {
  SubsampleRng rng;
  explicit rtlr_cu_rng(std::uint64_t seed) : rng(seed) {}
};
struct rtlr_cu_lr_basis {
  Problem* P = nullptr;
  std::unique_ptr<LowRankEngine> e;
  DBuf<double> sol, tmp;  // padded solution blocks (sharded all-gathers) and staging
};
struct rtlr_cu_inner {
  Problem* P = nullptr;
  std::unique_ptr<LowRankEngine> e;
  InnerResult r;
};

namespace {

LowRankParams params_of(const rtlr_cu_lr_params* o) {
  LowRankParams p;
  if (o) {
    p.p = o->p;
    p.q = o->q;
    p.eps_res = o->eps_res;
    p.eps_diff = o->eps_diff;
    p.eps_svd = o->eps_svd;
    p.eps_mgs = o->eps_mgs;
  }
  return p;
}

std::vector<int> ints(const int* a, int n) { return n > 0 ? std::vector<int>(a, a + n) : std::vector<int>(); }

void check_angles(const std::vector<int>& a, int nomega, const char* who) {
  for (int j : a)
    if (j < 0 || j >= nomega) throw std::invalid_argument(std::string(who) + ": angle index out of range");
}

// columns the engine writes for m items (sharded: the all-gather's padding)
int padded_cols(const Problem& P, int m) {
  if (P.nranks() <= 1 || !P.sharded()) return m;
  return shard_block(m, P.nranks(), P.rank()).bsz * P.nranks();
}

}  // namespace

extern "C" {

int rtlr_cu_problem_upload(const rtlr_cu_problem_desc* d, int device, rtlr_cu_problem** out) {
  return guard([&] {
    need(d && out, "problem_upload: null argument");
    ProblemArrays a;
    a.nx = d->nx;
    a.ny = d->ny;
    a.x_min = d->x_min;
    a.x_max = d->x_max;
    a.y_min = d->y_min;
    a.y_max = d->y_max;
    a.n_theta = d->n_theta;
    a.n_omega_z = d->n_omega_z;
    a.n_omega = d->n_omega;
    a.dirs = d->dirs;
    a.weights = d->weights;
    a.sigma_t = d->sigma_t_blocks;
    a.sigma_s = d->sigma_s_blocks;
    a.sigma_a = d->sigma_a_blocks;
    a.source = d->source;
    a.boundary = d->boundary;
    a.sip = d->sip_bsr;
    a.use_dsa = d->use_dsa != 0;
    HostProblem hp;
    assemble_arrays(a, hp);
    auto p = std::make_unique<rtlr_cu_problem>();
    p->p = std::make_unique<Problem>(std::move(hp), device);
    *out = p.release();
  });
}

void rtlr_cu_lr_params_default(rtlr_cu_lr_params* o) {
  if (!o) return;
  const LowRankParams d;
  o->p = d.p;
  o->q = d.q;
  o->eps_res = d.eps_res;
  o->eps_diff = d.eps_diff;
  o->eps_svd = d.eps_svd;
  o->eps_mgs = d.eps_mgs;
}

int rtlr_cu_rng_create(uint64_t seed, rtlr_cu_rng** out) {
  return guard([&] {
    need(out != nullptr, "rng: null argument");
    *out = new rtlr_cu_rng(seed);
  });
}

void rtlr_cu_rng_destroy(rtlr_cu_rng* r) { delete r; }

int rtlr_cu_rng_draw_below(rtlr_cu_rng* r, uint64_t n, uint64_t* out) {
  return guard([&] {
    need(r && out, "rng: null argument");
    *out = r->rng.draw_below(n);
  });
}

int rtlr_cu_rng_sample(rtlr_cu_rng* r, const int* pool, int n, int count, int* out, int* n_out) {
  return guard([&] {
    need(r && (pool || n == 0) && n >= 0 && out && n_out, "rng: bad argument");
    const std::vector<int> s = r->rng.sample_without_replacement(ints(pool, n), count);
    std::copy(s.begin(), s.end(), out);
    *n_out = static_cast<int>(s.size());
  });
}

int rtlr_cu_lr_basis_create(rtlr_cu_problem* p, const rtlr_cu_lr_params* params, const double* rhs_core, int where,
                            rtlr_cu_lr_basis** out) {
  return guard([&] {
    need(p && rhs_core && out, "LowRankBasis: null argument");
    Problem& P = gpu(p);
    auto b = std::make_unique<rtlr_cu_lr_basis>();
    b->P = &P;
    b->e = std::make_unique<LowRankEngine>(P, params_of(params));
    In r(rhs_core, P.host().ndof, where, P.stream());
    b->e->reset_rhs(r.d);
    RTLR_CUDA(cudaStreamSynchronize(P.stream()));
    *out = b.release();
  });
}

void rtlr_cu_lr_basis_destroy(rtlr_cu_lr_basis* b) { delete b; }

int rtlr_cu_lr_basis_info(const rtlr_cu_lr_basis* b, int64_t info[4]) {
  return guard([&] {
    need(b && info, "LowRankBasis: null argument");
    info[0] = b->e->rank();
    info[1] = b->e->snapshot_count();
    info[2] = b->e->n();
    info[3] = b->e->n_omega();
  });
}

int rtlr_cu_lr_basis_get(const rtlr_cu_lr_basis* b, const char* what, double* out, int where) {
  return guard([&] {
    need(b && what && out, "LowRankBasis: null argument");
    const LowRankEngine& e = *b->e;
    cudaStream_t s = e.stream();
    const std::string w = what;
    const long long r = e.rank(), n = e.n();
    auto copy2d = [&](const double* src, long long ld, long long rows, long long cols) {
      if (rows == 0 || cols == 0) return;
      RTLR_CUDA(cudaMemcpy2DAsync(out, rows * sizeof(double), src, ld * sizeof(double), rows * sizeof(double), cols,
                                  where == RTLR_CU_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
      RTLR_CUDA(cudaStreamSynchronize(s));
    };
    if (w == "basis") copy2d(e.X(), e.ldx(), n, r);
    else if (w == "record") copy2d(e.record(), e.ldr(), r, e.snapshot_count());
    else if (w == "dx_minus") copy2d(e.proj(0), e.ldp(), r, r);
    else if (w == "dx_plus") copy2d(e.proj(1), e.ldp(), r, r);
    else if (w == "dy_minus") copy2d(e.proj(2), e.ldp(), r, r);
    else if (w == "dy_plus") copy2d(e.proj(3), e.ldp(), r, r);
    else if (w == "sigma_t") copy2d(e.proj(4), e.ldp(), r, r);
    else if (w == "prhs") copy_out(out, e.prhs(), r, where, s);
    else if (w == "rhs_core") copy_out(out, e.rhs_core(), n, where, s);
    else throw std::invalid_argument("LowRankBasis: unknown quantity '" + w + "'");
  });
}

int rtlr_cu_lr_basis_sampled(const rtlr_cu_lr_basis* b, int* out) {
  return guard([&] {
    need(b && out, "LowRankBasis: null argument");
    std::copy(b->e->sampled().begin(), b->e->sampled().end(), out);
  });
}

int rtlr_cu_lr_mgs_ro_update(rtlr_cu_lr_basis* b, const double* snapshots, const int* angles, int n, double eps_mgs,
                             double drop_tol, int where, int* reorthogonalized) {
  return guard([&] {
    need(b && snapshots && angles && n >= 1, "mgs_ro_update: bad argument");
    LowRankEngine& e = *b->e;
    const std::vector<int> a = ints(angles, n);
    check_angles(a, e.n_omega(), "mgs_ro_update");
    In sn(snapshots, static_cast<size_t>(e.n()) * n, where, e.stream());
    e.set_eps_mgs(eps_mgs);
    e.set_drop_tol(drop_tol);
    const bool re = e.mgs_ro_update(sn.d, a);
    if (reorthogonalized) *reorthogonalized = re ? 1 : 0;
  });
}

int rtlr_cu_lr_update_projections(rtlr_cu_lr_basis* b, int reorthogonalized) {
  return guard([&] {
    need(b != nullptr, "update_projections: null argument");
    b->e->update_projections(reorthogonalized != 0);
    RTLR_CUDA(cudaStreamSynchronize(b->e->stream()));
  });
}

int rtlr_cu_lr_galerkin_solve(rtlr_cu_lr_basis* b, const int* angles, int m, double* sol, int where) {
  return guard([&] {
    need(b && angles && sol && m >= 0, "galerkin_solve: bad argument");
    LowRankEngine& e = *b->e;
    if (e.rank() < 1) throw std::runtime_error("galerkin_solve: empty basis");
    const std::vector<int> a = ints(angles, m);
    check_angles(a, e.n_omega(), "galerkin_solve");
    if (m == 0) return;
    const long long r = e.rank();
    double* d = b->sol.ensure(static_cast<size_t>(r) * padded_cols(*b->P, m));
    e.galerkin(a, d, r);
    e.check();  // the deferred non-finite flag: "galerkin_solve: singular reduced system"
    copy_out(sol, d, static_cast<size_t>(r) * m, where, e.stream());
  });
}

int rtlr_cu_lr_residual_norms(rtlr_cu_lr_basis* b, const int* angles, int m, const double* coeffs, double* norms,
                              int where) {
  return guard([&] {
    need(b && angles && coeffs && norms && m >= 0, "residual_norms: bad argument");
    LowRankEngine& e = *b->e;
    const std::vector<int> a = ints(angles, m);
    check_angles(a, e.n_omega(), "residual_norms");
    if (m == 0) return;
    In c(coeffs, static_cast<size_t>(e.rank()) * m, where, e.stream());
    const std::vector<double> v = e.residual_norms(a, c.d, e.rank());
    if (where == RTLR_CU_DEVICE) {
      RTLR_CUDA(cudaMemcpyAsync(norms, v.data(), m * sizeof(double), cudaMemcpyHostToDevice, e.stream()));
      RTLR_CUDA(cudaStreamSynchronize(e.stream()));
    } else {
      std::copy(v.begin(), v.end(), norms);
    }
  });
}

int rtlr_cu_lr_greedy_subsample(rtlr_cu_lr_basis* b, const unsigned char* sampled_mask, int p, int q, rtlr_cu_rng* rng,
                                int* selected, int* n_selected, double* max_residual, int* candidates,
                                int* n_candidates, double* candidate_solutions, double* residual_norms, int where) {
  return guard([&] {
    need(b && sampled_mask && rng && selected && n_selected && candidates && n_candidates,
         "greedy_subsample: null argument");
    if (p < 1 || q < p) throw std::invalid_argument("greedy_subsample: need 1 <= p <= q");
    LowRankEngine& e = *b->e;
    if (e.rank() < 1) throw std::runtime_error("galerkin_solve: empty basis");
    std::vector<char> mask(e.n_omega());
    for (int j = 0; j < e.n_omega(); ++j) mask[j] = sampled_mask[j] ? 1 : 0;
    const GreedyOutcome g = e.greedy_subsample(mask, p, q, rng->rng);
    std::copy(g.selected.begin(), g.selected.end(), selected);
    *n_selected = static_cast<int>(g.selected.size());
    std::copy(g.candidates.begin(), g.candidates.end(), candidates);
    *n_candidates = static_cast<int>(g.candidates.size());
    if (max_residual) *max_residual = g.max_residual;
    if (residual_norms) std::copy(g.residual_norms.begin(), g.residual_norms.end(), residual_norms);
    if (candidate_solutions)
      copy_out(candidate_solutions, e.cand_sol(), static_cast<size_t>(e.rank()) * g.candidates.size(), where,
               e.stream());
  });
}

int rtlr_cu_lr_build_coefficients(rtlr_cu_lr_basis* b, const int* candidates, int m, const double* candidate_solutions,
                                  double* C, double* phi, int where) {
  return guard([&] {
    need(b && m >= 0 && (m == 0 || (candidates && candidate_solutions)), "build_full_coefficients: bad argument");
    LowRankEngine& e = *b->e;
    if (e.rank() < 1) throw std::runtime_error("galerkin_solve: empty basis");
    const std::vector<int> cand = ints(candidates, m);
    check_angles(cand, e.n_omega(), "build_full_coefficients");
    In cs(candidate_solutions, static_cast<size_t>(e.rank()) * m, where, e.stream());
    e.build_full_coefficients(m > 0 ? &cand : nullptr, cs.d);
    e.phi_from_C();
    e.check();
    if (C) copy_out(C, e.C(), static_cast<size_t>(e.rank()) * e.n_omega(), where, e.stream());
    if (phi) copy_out(phi, e.phi(), e.n(), where, e.stream());
  });
}

int rtlr_cu_truncation_rank(const double* s, int n, double eps_svd, int* out) {
  return guard([&] {
    need((s || n == 0) && n >= 0 && out, "truncation_rank: bad argument");
    *out = truncation_rank(std::vector<double>(s, s + n), eps_svd);
  });
}

int rtlr_cu_truncate_factors(rtlr_cu_problem* p, const double* C, const double* X, int rank, double eps_svd, int where,
                             int* rank_out, double* X_out, double* S_out, double* V_out) {
  return guard([&] {
    need(p && C && X && rank >= 1 && rank_out && S_out, "truncate_factors: bad argument");
    Problem& P = gpu(p);
    const size_t n = P.host().ndof, nom = P.host().n_omega;
    LowRankEngine e(P, LowRankParams{});
    In c(C, static_cast<size_t>(rank) * nom, where, P.stream()), x(X, n * rank, where, P.stream());
    e.load_factors(c.d, x.d, rank);
    const std::vector<double> sv = e.svd(false, 0, nullptr, nullptr);
    if (!X_out && !V_out) {  // singular values only
      *rank_out = static_cast<int>(sv.size());
      std::copy(sv.begin(), sv.end(), S_out);
      return;
    }
    need(X_out && V_out, "truncate_factors: X_out and V_out go together");
    const int r = truncation_rank(sv, eps_svd);
    std::vector<double> Xo, Vo;
    const std::vector<double> s2 = e.svd(true, r, &Xo, &Vo);
    *rank_out = r;
    std::copy(s2.begin(), s2.begin() + r, S_out);
    if (where == RTLR_CU_DEVICE) {
      RTLR_CUDA(cudaMemcpyAsync(X_out, Xo.data(), Xo.size() * sizeof(double), cudaMemcpyHostToDevice, P.stream()));
      RTLR_CUDA(cudaMemcpyAsync(V_out, Vo.data(), Vo.size() * sizeof(double), cudaMemcpyHostToDevice, P.stream()));
      RTLR_CUDA(cudaStreamSynchronize(P.stream()));
    } else {
      std::copy(Xo.begin(), Xo.end(), X_out);
      std::copy(Vo.begin(), Vo.end(), V_out);
    }
  });
}

int rtlr_cu_low_rank_si(rtlr_cu_problem* p, const double* phi_prev, const rtlr_cu_lr_params* params, rtlr_cu_rng* rng,
                        int where, rtlr_cu_inner** out) {
  return guard([&] {
    need(p && phi_prev && rng && out, "low_rank_si: null argument");
    Problem& P = gpu(p);
    auto r = std::make_unique<rtlr_cu_inner>();
    r->P = &P;
    r->e = std::make_unique<LowRankEngine>(P, params_of(params));
    In ph(phi_prev, P.host().ndof, where, P.stream());
    r->r = r->e->inner(ph.d, rng->rng);
    *out = r.release();
  });
}

int rtlr_cu_inner_info(const rtlr_cu_inner* r, int64_t info[8]) {
  return guard([&] {
    need(r && info, "inner: null argument");
    info[0] = r->r.iterations;
    info[1] = r->r.rank;
    info[2] = r->r.sampled_count;
    info[3] = r->r.reorthogonalizations;
    info[4] = r->r.verification_rejections;
    info[5] = r->r.exhausted ? 1 : 0;
    info[6] = r->e->n();
    info[7] = r->e->n_omega();
  });
}

int rtlr_cu_inner_get(const rtlr_cu_inner* r, const char* what, double* out, int where) {
  return guard([&] {
    need(r && what && out, "inner: null argument");
    LowRankEngine& e = *r->e;
    const std::string w = what;
    const long long rk = e.rank(), n = e.n();
    if (w == "phi_star") {
      copy_out(out, e.phi(), n, where, e.stream());
    } else if (w == "coefficients") {
      copy_out(out, e.C(), static_cast<size_t>(rk) * e.n_omega(), where, e.stream());
    } else if (w == "basis") {
      if (rk == 0) return;
      RTLR_CUDA(cudaMemcpy2DAsync(out, n * sizeof(double), e.X(), e.ldx() * sizeof(double), n * sizeof(double), rk,
                                  where == RTLR_CU_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                                  e.stream()));
      RTLR_CUDA(cudaStreamSynchronize(e.stream()));
    } else {
      throw std::invalid_argument("inner: unknown quantity '" + w + "'");
    }
  });
}

int rtlr_cu_inner_sampled(const rtlr_cu_inner* r, int* out) {
  return guard([&] {
    need(r && out, "inner: null argument");
    std::copy(r->r.sampled_order.begin(), r->r.sampled_order.end(), out);
  });
}

void rtlr_cu_inner_destroy(rtlr_cu_inner* r) { delete r; }

}  // extern "C"
