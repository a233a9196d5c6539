// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp header).
// Restates proj/src/diffusion.cpp, proj/src/full_rank.cpp,
// proj/src/low_rank.cpp and proj/src/report.cpp:47-74.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <numeric>

#include "oracle.hpp"

namespace oracle {

// ============================================================ diffusion
namespace {

// proj/src/diffusion.cpp:15-28
Mat stiffness_matrix_1d(int degree, double h) {
  int n = degree + 1;
  GaussLegendre gl = gauss_legendre(degree + 2);
  Mat st(n, n);
  for (int g = 0; g < static_cast<int>(gl.nodes.size()); ++g) {
    Vec dphi(n);
    for (int m = 0; m < n; ++m)
      dphi[m] = std::sqrt((2.0 * m + 1.0) / h) * legendre_derivative(m, gl.nodes[g]) * 2.0 / h;
    const double alpha = 0.5 * h * gl.weights[g];
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) st(i, j) += (alpha * dphi[i]) * dphi[j];
  }
  return st;
}
// proj/src/diffusion.cpp:30-48
Vec edge_values(int degree, double h, bool right) {
  Vec v(degree + 1);
  for (int m = 0; m <= degree; ++m) {
    double p = right ? 1.0 : ((m % 2 == 0) ? 1.0 : -1.0);
    v[m] = std::sqrt((2.0 * m + 1.0) / h) * p;
  }
  return v;
}
Vec edge_derivatives(int degree, double h, bool right) {
  Vec v(degree + 1);
  for (int m = 0; m <= degree; ++m) {
    double dp = 0.5 * m * (m + 1.0);
    if (!right && m % 2 == 0) dp = -dp;
    v[m] = std::sqrt((2.0 * m + 1.0) / h) * dp * 2.0 / h;
  }
  return v;
}
Mat tx(const Mat& bx, int degree) {
  int n = degree + 1, s = n * n;
  Mat out(s, s);
  for (int my = 0; my < n; ++my)
    for (int mx = 0; mx < n; ++mx)
      for (int lx = 0; lx < n; ++lx) out(my * n + mx, my * n + lx) = bx(mx, lx);
  return out;
}
Mat ty(const Mat& by, int degree) {
  int n = degree + 1, s = n * n;
  Mat out(s, s);
  for (int mx = 0; mx < n; ++mx)
    for (int my = 0; my < n; ++my)
      for (int ly = 0; ly < n; ++ly) out(my * n + mx, ly * n + mx) = by(my, ly);
  return out;
}
void append(std::vector<Triplet>& t, int r0, int c0, const Mat& blk) {
  for (int i = 0; i < blk.rows; ++i)
    for (int j = 0; j < blk.cols; ++j)
      if (blk(i, j) != 0.0) t.push_back({r0 + i, c0 + j, blk(i, j)});
}
// proj/src/diffusion.cpp:79-88
Mat sip_face(const Vec& vt, const Vec& gt, double st, const Vec& vu, const Vec& gu, double su,
             double gamma) {
  int n = static_cast<int>(vt.size());
  Mat e(n, n);
  for (int k = 0; k < n; ++k)
    for (int l = 0; l < n; ++l)
      e(k, l) = -gu[l] * st * vt[k] - gt[k] * su * vu[l] + gamma * st * su * vt[k] * vu[l];
  return e;
}
Vec scaled(double a, const Vec& v) {
  Vec o(v.size());
  for (size_t i = 0; i < v.size(); ++i) o[i] = a * v[i];
  return o;
}

}  // namespace

// proj/src/diffusion.cpp:90-201 (assembly identical; SimplicialLDLT replaced
// by a banded LDL^T in natural DOF order, bandwidth s*(nx+1)-1).
DiffusionSystem::DiffusionSystem(const DGSpace& space, const DiscreteOperators& ops, bool factor) {
  const SpatialMesh& mesh = space.mesh;
  const int k = space.degree, s = space.dofs_per_cell(), n = space.size();
  const double dx = mesh.dx(), dy = mesh.dy();
  const double pen = 4.0 * std::max(k * (k + 1), 1);
  std::vector<double> d_cell(mesh.cell_count());
  for (int c = 0; c < mesh.cell_count(); ++c) {
    double sig = ops.sigma_t_blocks[c](0, 0);
    if (!(sig > 0.0)) throw std::runtime_error("build_diffusion: sigma_t must be positive");
    d_cell[c] = 1.0 / (3.0 * sig);
  }
  Mat stx = stiffness_matrix_1d(k, dx), sty = stiffness_matrix_1d(k, dy);
  Mat vol = tx(stx, k), voly = ty(sty, k);
  for (size_t i = 0; i < vol.a.size(); ++i) vol.a[i] += voly.a[i];
  Vec vxl = edge_values(k, dx, false), vxr = edge_values(k, dx, true);
  Vec gxl = edge_derivatives(k, dx, false), gxr = edge_derivatives(k, dx, true);
  Vec vyl = edge_values(k, dy, false), vyr = edge_values(k, dy, true);
  Vec gyl = edge_derivatives(k, dy, false), gyr = edge_derivatives(k, dy, true);

  std::vector<Triplet> trips;
  for (int c = 0; c < mesh.cell_count(); ++c) {
    Mat blk(s, s);
    for (size_t i = 0; i < blk.a.size(); ++i) blk.a[i] = d_cell[c] * vol.a[i];
    append(trips, c * s, c * s, blk);
  }
  for (int b = 0; b < mesh.ny; ++b)
    for (int af = 0; af <= mesh.nx; ++af) {
      bool has_l = af > 0, has_r = af < mesh.nx;
      int cl = has_l ? mesh.cell_index(af - 1, b) : -1;
      int cr = has_r ? mesh.cell_index(af, b) : -1;
      if (has_l && has_r) {
        double dl = d_cell[cl], dr = d_cell[cr];
        double wsum = dl + dr, wl = dr / wsum, wr = dl / wsum;
        double dharm = 2.0 * dl * dr / wsum;
        double gamma = pen * dharm / dx;
        Vec fl = scaled(wl * dl, gxr), fr = scaled(wr * dr, gxl);
        append(trips, cl * s, cl * s, tx(sip_face(vxr, fl, 1, vxr, fl, 1, gamma), k));
        append(trips, cl * s, cr * s, tx(sip_face(vxr, fl, 1, vxl, fr, -1, gamma), k));
        append(trips, cr * s, cl * s, tx(sip_face(vxl, fr, -1, vxr, fl, 1, gamma), k));
        append(trips, cr * s, cr * s, tx(sip_face(vxl, fr, -1, vxl, fr, -1, gamma), k));
      } else {
        int c = has_l ? cl : cr;
        const Vec& v = has_l ? vxr : vxl;
        Vec g = has_l ? scaled(d_cell[c], gxr) : scaled(-d_cell[c], gxl);
        double gamma = pen * d_cell[c] / dx;
        append(trips, c * s, c * s, tx(sip_face(v, g, 1, v, g, 1, gamma), k));
      }
    }
  for (int a = 0; a < mesh.nx; ++a)
    for (int bf = 0; bf <= mesh.ny; ++bf) {
      bool has_b = bf > 0, has_t = bf < mesh.ny;
      int cb = has_b ? mesh.cell_index(a, bf - 1) : -1;
      int ct = has_t ? mesh.cell_index(a, bf) : -1;
      if (has_b && has_t) {
        double db = d_cell[cb], dt = d_cell[ct];
        double wsum = db + dt, wb = dt / wsum, wt = db / wsum;
        double dharm = 2.0 * db * dt / wsum;
        double gamma = pen * dharm / dy;
        Vec fb = scaled(wb * db, gyr), ft = scaled(wt * dt, gyl);
        append(trips, cb * s, cb * s, ty(sip_face(vyr, fb, 1, vyr, fb, 1, gamma), k));
        append(trips, cb * s, ct * s, ty(sip_face(vyr, fb, 1, vyl, ft, -1, gamma), k));
        append(trips, ct * s, cb * s, ty(sip_face(vyl, ft, -1, vyr, fb, 1, gamma), k));
        append(trips, ct * s, ct * s, ty(sip_face(vyl, ft, -1, vyl, ft, -1, gamma), k));
      } else {
        int c = has_b ? cb : ct;
        const Vec& v = has_b ? vyr : vyl;
        Vec g = has_b ? scaled(d_cell[c], gyr) : scaled(-d_cell[c], gyl);
        double gamma = pen * d_cell[c] / dy;
        append(trips, c * s, c * s, ty(sip_face(v, g, 1, v, g, 1, gamma), k));
      }
    }
  a_diff_ = csr_add(csr_from_triplets(n, trips), ops.sigma_a);
  sigma_s_ = ops.sigma_s;
  if (!factor) return;

  // Banded LDL^T.
  n_ = n;
  bw_ = s * (mesh.nx + 1) - 1;
  const int w = bw_ + 1;
  band_.assign(static_cast<size_t>(n) * w, 0.0);
  auto B = [&](int i, int j) -> double& { return band_[static_cast<size_t>(i) * w + (j - i + bw_)]; };
  for (int i = 0; i < n; ++i)
    for (int kk = a_diff_.rowptr[i]; kk < a_diff_.rowptr[i + 1]; ++kk) {
      int j = a_diff_.colidx[kk];
      if (j <= i) B(i, j) = a_diff_.val[kk];
    }
  std::vector<double> wrow(w);
  for (int i = 0; i < n; ++i) {
    const int j0 = std::max(0, i - bw_);
    for (int j = j0; j < i; ++j) {
      double sacc = B(i, j);
      const int k0 = std::max(j0, j - bw_);
      for (int kk = k0; kk < j; ++kk) sacc -= wrow[kk - j0] * B(j, kk);
      wrow[j - j0] = sacc;            // L(i,j) * D(j)
      B(i, j) = sacc / B(j, j);       // L(i,j)
    }
    double d = B(i, i);
    for (int j = j0; j < i; ++j) d -= wrow[j - j0] * B(i, j);
    if (!(d > 0.0))
      throw std::runtime_error("build_diffusion: factorization failed (matrix not positive definite)");
    B(i, i) = d;
  }
}

Vec DiffusionSystem::solve(const Vec& rhs) const {
  if (band_.empty()) throw std::runtime_error("diffusion solve failed (matrix not factored)");
  const int w = bw_ + 1;
  auto B = [&](int i, int j) { return band_[static_cast<size_t>(i) * w + (j - i + bw_)]; };
  Vec x = rhs;
  for (int i = 0; i < n_; ++i) {
    double sacc = x[i];
    for (int j = std::max(0, i - bw_); j < i; ++j) sacc -= B(i, j) * x[j];
    x[i] = sacc;
  }
  for (int i = 0; i < n_; ++i) x[i] /= B(i, i);
  for (int i = n_ - 1; i >= 0; --i) {
    const double xi = x[i];
    for (int j = std::max(0, i - bw_); j < i; ++j) x[j] -= B(i, j) * xi;
  }
  for (double v : x)
    if (!std::isfinite(v)) throw std::runtime_error("diffusion solve failed");
  return x;
}

// proj/src/diffusion.cpp:210-213
Vec DiffusionSystem::correct(const Vec& phi_star, const Vec& phi_prev) const {
  Vec d(phi_star.size());
  for (size_t i = 0; i < d.size(); ++i) d[i] = phi_star[i] - phi_prev[i];
  return solve(sigma_s_.mul(d));
}

// ============================================================ full rank
// proj/src/full_rank.cpp:11-39
BoundaryData build_boundary_data(const DGSpace& space, const AngularQuadrature& quad,
                                 const Field& g) {
  BoundaryData bc;
  const SpatialMesh& mesh = space.mesh;
  const int nq = space.degree + 2;
  GaussLegendre gl = gauss_legendre(nq);
  double max_abs = 0.0;
  for (int b = 0; b < mesh.ny; ++b)
    for (int q = 0; q < nq; ++q) {
      double y = mesh.y_center(b) + 0.5 * mesh.dy() * gl.nodes[q];
      max_abs = std::max(max_abs, std::abs(g(mesh.x_min, y)));
      max_abs = std::max(max_abs, std::abs(g(mesh.x_max, y)));
    }
  for (int a = 0; a < mesh.nx; ++a)
    for (int q = 0; q < nq; ++q) {
      double x = mesh.x_center(a) + 0.5 * mesh.dx() * gl.nodes[q];
      max_abs = std::max(max_abs, std::abs(g(x, mesh.y_min)));
      max_abs = std::max(max_abs, std::abs(g(x, mesh.y_max)));
    }
  if (max_abs == 0.0) return bc;
  bc.any = true;
  bc.per_angle.resize(quad.size());
  for (int j = 0; j < quad.size(); ++j) bc.per_angle[j] = boundary_vector(space, quad, g, j);
  return bc;
}

namespace {
Vec rhs_core_of(const DiscreteOperators& ops, const Vec& phi, const Vec& source) {
  Vec r = ops.sigma_s.mul(phi);
  for (size_t i = 0; i < r.size(); ++i) r[i] += source[i];
  return r;
}
Vec with_bc(const Vec& rhs_core, const BoundaryData& bc, int j) {
  Vec r = rhs_core;
  if (const Vec* g = bc.get(j))
    for (size_t i = 0; i < r.size(); ++i) r[i] += (*g)[i];
  return r;
}
// psi * w (Eigen GEMV, column-major): accumulate column by column.
Vec mat_vec(const Mat& m, const Vec& w) {
  Vec y(m.rows, 0.0);
  for (int j = 0; j < m.cols; ++j) {
    const double* c = m.col(j);
    for (int i = 0; i < m.rows; ++i) y[i] += c[i] * w[j];
  }
  return y;
}
}  // namespace

// proj/src/full_rank.cpp:41-58
SIStepResult si_step(const DiscreteOperators& ops, const AngularQuadrature& quad,
                     const BoundaryData& bc, const Vec& source, const Vec& phi_prev) {
  const int n = ops.space.size(), n_omega = quad.size();
  Vec rhs_core = rhs_core_of(ops, phi_prev, source);
  SIStepResult out;
  out.psi = Mat(n, n_omega);
  for (int j = 0; j < n_omega; ++j) {
    Vec psi = sweep(ops, quad, j, with_bc(rhs_core, bc, j));
    std::copy(psi.begin(), psi.end(), out.psi.col(j));
  }
  out.phi_star = mat_vec(out.psi, quad.weights);
  return out;
}

// proj/src/full_rank.cpp:60-122
SolveReport solve_full_rank(const DiscreteOperators& ops, const AngularQuadrature& quad,
                            const BoundaryData& bc, const Vec& source,
                            const DiffusionSystem* dsa, const FullRankOptions& opts) {
  if (opts.use_dsa && dsa == nullptr)
    throw std::invalid_argument("solve_full_rank: DSA requested but no diffusion system");
  const int n = ops.space.size(), n_omega = quad.size();
  SolveReport report;
  report.method = "full";
  report.psi_dofs = static_cast<long long>(n) * n_omega;
  auto t0 = std::chrono::steady_clock::now();
  Vec phi(n, 0.0), phi_star;
  Mat psi;
  for (int it = 1; it <= opts.max_iterations; ++it) {
    Vec rhs_core = rhs_core_of(ops, phi, source);
    if (opts.store_psi) {
      if (psi.a.empty()) psi = Mat(n, n_omega);
      for (int j = 0; j < n_omega; ++j) {
        Vec col = sweep(ops, quad, j, with_bc(rhs_core, bc, j));
        std::copy(col.begin(), col.end(), psi.col(j));
      }
      phi_star = mat_vec(psi, quad.weights);
    } else {
      phi_star.assign(n, 0.0);
      for (int j = 0; j < n_omega; ++j) {
        Vec col = sweep(ops, quad, j, with_bc(rhs_core, bc, j));
        for (int i = 0; i < n; ++i) phi_star[i] += quad.weights[j] * col[i];
      }
    }
    Vec d(n);
    for (int i = 0; i < n; ++i) d[i] = phi_star[i] - phi[i];
    OuterRecord rec;
    rec.diff_two_norm = norm2(d);
    rec.diff_inf_norm = norm_inf(d);
    report.history.push_back(rec);
    report.iterations = it;
    if (rec.diff_inf_norm <= opts.eps_si_sa) {
      report.converged = true;
      phi = phi_star;
      break;
    }
    if (opts.use_dsa) {
      Vec delta = dsa->correct(phi_star, phi);
      for (int i = 0; i < n; ++i) phi[i] = phi_star[i] + delta[i];
    } else {
      phi = phi_star;
    }
  }
  if (!report.converged) phi = phi_star;
  report.solve_seconds =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  report.phi = phi;
  if (opts.store_psi) {
    report.has_psi = true;
    report.psi = std::move(psi);
  }
  return report;
}

// ============================================================ low rank
// proj/src/low_rank.cpp:15-37 (mt19937_64 + masked rejection)
std::uint64_t SubsampleRng::draw_below(std::uint64_t n) {
  if (n == 0) throw std::invalid_argument("draw_below: empty range");
  std::uint64_t mask = ~std::uint64_t{0};
  std::uint64_t limit = n - 1;
  int bits = 0;
  while (bits < 64 && (limit >> bits)) ++bits;
  mask = (bits >= 64) ? mask : ((std::uint64_t{1} << bits) - 1);
  std::uint64_t v;
  do {
    v = engine_() & mask;
  } while (v >= n);
  return v;
}

std::vector<int> SubsampleRng::sample_without_replacement(std::vector<int> pool, int count) {
  count = std::min<int>(count, static_cast<int>(pool.size()));
  for (int i = 0; i < count; ++i) {
    int j = i + static_cast<int>(draw_below(pool.size() - i));
    std::swap(pool[i], pool[j]);
  }
  pool.resize(count);
  return pool;
}

// proj/src/low_rank.cpp:39-43
LowRankBasis::LowRankBasis(const DiscreteOperators& ops, const AngularQuadrature& quad,
                           const BoundaryData& bc, Vec rhs_core)
    : ops_(&ops), quad_(&quad), bc_(&bc), rhs_core_(std::move(rhs_core)), proj_(5) {}

double& LowRankBasis::P(int k, int i, int j) { return proj_[k][j][i]; }

Mat LowRankBasis::basis() const {
  const int n = ops_->space.size();
  Mat x(n, rank_);
  for (int j = 0; j < rank_; ++j) std::copy(x_[j].begin(), x_[j].end(), x.col(j));
  return x;
}

Mat LowRankBasis::coefficient_record() const {
  Mat r(rank_, n_snap_);
  for (int j = 0; j < n_snap_; ++j)
    for (int i = 0; i < rank_ && i < static_cast<int>(rec_[j].size()); ++i) r(i, j) = rec_[j][i];
  return r;
}

Mat LowRankBasis::projected(int k) const {
  Mat m(rank_, rank_);
  for (int j = 0; j < rank_; ++j)
    for (int i = 0; i < rank_; ++i) m(i, j) = proj_[k][j][i];
  return m;
}

// proj/src/low_rank.cpp:66-132: CGS per snapshot, conditional second pass,
// drop test, overlap-triggered Householder rebuild.
bool LowRankBasis::mgs_ro_update(const Mat& snaps, const std::vector<int>& angles,
                                 double eps_mgs, double drop_tol) {
  const int n = ops_->space.size();
  const int p_in = snaps.cols;
  if (static_cast<int>(angles.size()) != p_in)
    throw std::invalid_argument("mgs_ro_update: angle/snapshot count mismatch");
  prev_rank_ = rank_;
  const int m0 = n_snap_;
  std::vector<Vec> accepted;
  for (int i = 0; i < p_in; ++i) {
    const double* snap = snaps.col(i);
    Vec rem(snap, snap + n);
    const double norm0 = norm2(rem);
    Vec chat;
    if (rank_ > 0) {
      chat.assign(rank_, 0.0);
      for (int k = 0; k < rank_; ++k) chat[k] = dot(x_[k].data(), snap, n);
      for (int k = 0; k < rank_; ++k)
        for (int t = 0; t < n; ++t) rem[t] -= x_[k][t] * chat[k];
      if (norm2(rem) < 0.5 * norm0) {
        Vec corr(rank_);
        for (int k = 0; k < rank_; ++k) corr[k] = dot(x_[k].data(), rem.data(), n);
        for (int k = 0; k < rank_; ++k)
          for (int t = 0; t < n; ++t) rem[t] -= x_[k][t] * corr[k];
        for (int k = 0; k < rank_; ++k) chat[k] += corr[k];
      }
    }
    Vec reccol(rank_ + 1, 0.0);
    for (int k = 0; k < rank_; ++k) reccol[k] = chat[k];
    const double h = norm2(rem);
    if (norm0 > 0.0 && h > drop_tol * norm0) {
      for (int t = 0; t < n; ++t) rem[t] /= h;
      x_.push_back(std::move(rem));
      reccol[rank_] = h;
      accepted.emplace_back(snap, snap + n);
      ++rank_;
    } else {
      reccol.resize(rank_);
    }
    rec_.push_back(std::move(reccol));
    sampled_.push_back(angles[i]);
    ++n_snap_;
  }
  bool reorth = false;
  if (rank_ > prev_rank_ && rank_ >= 2) {
    const double overlap = std::abs(dot(x_[0].data(), x_[rank_ - 1].data(), n));
    reorth = overlap > eps_mgs;
  }
  if (reorth) {
    const int n_acc = static_cast<int>(accepted.size());
    const int r_new = prev_rank_ + n_acc;
    Mat m(n, r_new);
    for (int k = 0; k < prev_rank_; ++k) std::copy(x_[k].begin(), x_[k].end(), m.col(k));
    for (int k = 0; k < n_acc; ++k) std::copy(accepted[k].begin(), accepted[k].end(), m.col(prev_rank_ + k));
    Mat q, r;
    householder_qr(m, q, r);
    // old record (prev_rank x m0)
    std::vector<Vec> old(m0, Vec(prev_rank_, 0.0));
    for (int j = 0; j < m0; ++j)
      for (int i = 0; i < prev_rank_ && i < static_cast<int>(rec_[j].size()); ++i) old[j][i] = rec_[j][i];
    rank_ = r_new;
    for (int j = 0; j < n_snap_; ++j) rec_[j].assign(rank_, 0.0);
    if (m0 > 0 && prev_rank_ > 0)
      for (int j = 0; j < m0; ++j)
        for (int i = 0; i < rank_; ++i) {
          double acc = 0.0;
          for (int k = 0; k < prev_rank_; ++k) acc += r(i, k) * old[j][k];
          rec_[j][i] = acc;
        }
    for (int j = 0; j < p_in; ++j)
      for (int i = 0; i < rank_; ++i) rec_[m0 + j][i] = dot(q.col(i), snaps.col(j), n);
    x_.resize(rank_);
    for (int k = 0; k < rank_; ++k) x_[k].assign(q.col(k), q.col(k) + n);
  }
  return reorth;
}

// proj/src/low_rank.cpp:136-174 (border extension / direct reprojection)
void LowRankBasis::update_projections(bool reorth) {
  const int n = ops_->space.size();
  const Csr* mats[5] = {&ops_->d_x_minus, &ops_->d_x_plus, &ops_->d_y_minus, &ops_->d_y_plus,
                        &ops_->sigma_t};
  for (auto& pm : proj_) {
    pm.resize(rank_);
    for (auto& c : pm) c.resize(rank_, 0.0);
  }
  prhs_.resize(rank_, 0.0);
  if (!reorth) {
    const int p_new = rank_ - prev_rank_;
    if (p_new <= 0) return;
    const int r0 = prev_rank_;
    for (int k = 0; k < 5; ++k) {
      for (int j = 0; j < p_new; ++j) {
        const Vec& pj = x_[r0 + j];
        Vec ap = mats[k]->mul(pj);
        Vec atp = mats[k]->tmul(pj);
        for (int i = 0; i < r0; ++i) {
          P(k, i, r0 + j) = dot(x_[i].data(), ap.data(), n);
          P(k, r0 + j, i) = dot(atp.data(), x_[i].data(), n);
        }
        for (int i = 0; i < p_new; ++i) P(k, r0 + i, r0 + j) = dot(x_[r0 + i].data(), ap.data(), n);
      }
    }
    for (int j = 0; j < p_new; ++j) prhs_[r0 + j] = dot(x_[r0 + j].data(), rhs_core_.data(), n);
    return;
  }
  for (int k = 0; k < 5; ++k)
    for (int j = 0; j < rank_; ++j) {
      Vec ax = mats[k]->mul(x_[j]);
      for (int i = 0; i < rank_; ++i) P(k, i, j) = dot(x_[i].data(), ax.data(), n);
    }
  for (int i = 0; i < rank_; ++i) prhs_[i] = dot(x_[i].data(), rhs_core_.data(), n);
}

// proj/src/low_rank.cpp:176-183
Mat LowRankBasis::reduced_streaming(int angle) const {
  const double omx = quad_->omega_x(angle), omy = quad_->omega_y(angle);
  const auto& px = proj_[omx >= 0.0 ? 0 : 1];
  const auto& py = proj_[omy >= 0.0 ? 2 : 3];
  const auto& pt = proj_[4];
  Mat a(rank_, rank_);
  for (int j = 0; j < rank_; ++j)
    for (int i = 0; i < rank_; ++i) a(i, j) = omx * px[j][i] + omy * py[j][i] + pt[j][i];
  return a;
}

// proj/src/low_rank.cpp:185-190
Vec LowRankBasis::reduced_rhs(int angle) const {
  Vec r(prhs_.begin(), prhs_.begin() + rank_);
  if (const Vec* g = bc_->get(angle))
    for (int k = 0; k < rank_; ++k) r[k] += dot(x_[k].data(), g->data(), static_cast<int>(g->size()));
  return r;
}

// proj/src/low_rank.cpp:192-200
Vec LowRankBasis::galerkin_solve(int angle) const {
  if (rank_ < 1) throw std::runtime_error("galerkin_solve: empty basis");
  LU lu;
  lu.compute(reduced_streaming(angle));
  Vec c = lu.solve(reduced_rhs(angle));
  for (double v : c)
    if (!std::isfinite(v)) throw std::runtime_error("galerkin_solve: singular reduced system");
  return c;
}

Vec LowRankBasis::expand(const Vec& c) const {
  const int n = ops_->space.size();
  Vec y(n, 0.0);
  for (int k = 0; k < rank_; ++k)
    for (int t = 0; t < n; ++t) y[t] += x_[k][t] * c[k];
  return y;
}

// proj/src/low_rank.cpp:210-215
double LowRankBasis::residual_in_full_space(int angle, const Vec& y) const {
  StreamingOperator op = upwind_combination(*ops_, *quad_, angle);
  Vec ay = op.apply(y);
  Vec r(y.size());
  for (size_t i = 0; i < r.size(); ++i) r[i] = rhs_core_[i] - ay[i];
  if (const Vec* g = bc_->get(angle))
    for (size_t i = 0; i < r.size(); ++i) r[i] += (*g)[i];
  return norm2(r);
}

// proj/src/low_rank.cpp:217-252
SubsampleOutcome greedy_subsample(const LowRankBasis& basis, const std::vector<char>& mask, int p,
                                  int q, SubsampleRng& rng) {
  std::vector<int> pool;
  for (int j = 0; j < static_cast<int>(mask.size()); ++j)
    if (!mask[j]) pool.push_back(j);
  SubsampleOutcome out;
  if (pool.empty()) return out;
  out.candidates = rng.sample_without_replacement(std::move(pool), q);
  const int m = static_cast<int>(out.candidates.size());
  out.candidate_solutions.resize(m);
  out.residual_norms.resize(m);
  for (int i = 0; i < m; ++i) out.candidate_solutions[i] = basis.galerkin_solve(out.candidates[i]);
  for (int i = 0; i < m; ++i)
    out.residual_norms[i] =
        basis.residual_in_full_space(out.candidates[i], basis.expand(out.candidate_solutions[i]));
  std::vector<int> order(m);
  std::iota(order.begin(), order.end(), 0);
  std::sort(order.begin(), order.end(), [&](int a, int b) {
    if (out.residual_norms[a] != out.residual_norms[b])
      return out.residual_norms[a] > out.residual_norms[b];
    return out.candidates[a] < out.candidates[b];
  });
  out.max_residual = out.residual_norms[order.front()];
  const int take = std::min(p, m);
  for (int i = 0; i < take; ++i) out.selected.push_back(out.candidates[order[i]]);
  return out;
}

// proj/src/low_rank.cpp:254-266
int truncation_rank(const Vec& s, double eps_svd) {
  const int n = static_cast<int>(s.size());
  if (n == 0) return 0;
  double total = 0.0;
  for (double v : s) total += v;
  if (!(total > 0.0)) return 1;
  const double tol = eps_svd * total;
  double tail = 0.0;
  for (int i = n - 1; i >= 0; --i) {
    tail += s[i];
    if (tail > tol) return i + 1;
  }
  return 1;
}

// proj/src/low_rank.cpp:268-277
LowRankFactors truncate_factors(const Mat& c, const Mat& basis, double eps_svd) {
  Mat u, v;
  Vec s;
  svd_thin(c, &u, s, &v);
  const int r = truncation_rank(s, eps_svd);
  LowRankFactors f;
  f.S.assign(s.begin(), s.begin() + r);
  f.X = Mat(basis.rows, r);
  for (int j = 0; j < r; ++j)
    for (int k = 0; k < basis.cols; ++k) {
      const double ukj = u(k, j);
      const double* bk = basis.col(k);
      double* xj = f.X.col(j);
      for (int i = 0; i < basis.rows; ++i) xj[i] += bk[i] * ukj;
    }
  f.V = Mat(v.rows, r);
  for (int j = 0; j < r; ++j) std::copy(v.col(j), v.col(j) + v.rows, f.V.col(j));
  return f;
}

namespace {
// proj/src/low_rank.cpp:283-307 (blocks of 128 angles)
std::vector<double> batched_residual_norms(const LowRankBasis& basis, const std::vector<int>& angles,
                                           const Mat& coeffs) {
  std::vector<double> norms(angles.size());
  for (size_t i = 0; i < angles.size(); ++i) {
    const int j = angles[i];
    Vec c(coeffs.col(j), coeffs.col(j) + coeffs.rows);
    norms[i] = basis.residual_in_full_space(j, basis.expand(c));
  }
  return norms;
}
// proj/src/low_rank.cpp:311-336
Mat build_full_coefficients(const LowRankBasis& basis, const std::vector<char>& mask,
                            const SubsampleOutcome* reuse) {
  const int n_omega = static_cast<int>(mask.size());
  const int r = basis.rank();
  Mat c(r, n_omega);
  std::vector<char> done(n_omega, 0);
  const auto& angles = basis.sampled_angles();
  Mat rec = basis.coefficient_record();
  for (int i = 0; i < static_cast<int>(angles.size()); ++i) {
    std::copy(rec.col(i), rec.col(i) + r, c.col(angles[i]));
    done[angles[i]] = 1;
  }
  if (reuse)
    for (size_t i = 0; i < reuse->candidates.size(); ++i) {
      int j = reuse->candidates[i];
      if (!done[j]) {
        std::copy(reuse->candidate_solutions[i].begin(), reuse->candidate_solutions[i].end(), c.col(j));
        done[j] = 1;
      }
    }
  for (int j = 0; j < n_omega; ++j)
    if (!done[j]) {
      Vec g = basis.galerkin_solve(j);
      std::copy(g.begin(), g.end(), c.col(j));
    }
  return c;
}
Vec phi_from(const LowRankBasis& basis, const Mat& c, const Vec& w) {
  Vec cw(c.rows, 0.0);
  for (int j = 0; j < c.cols; ++j)
    for (int i = 0; i < c.rows; ++i) cw[i] += c(i, j) * w[j];
  return basis.expand(cw);
}
}  // namespace

// proj/src/low_rank.cpp:340-434
InnerLoopResult low_rank_si(const DiscreteOperators& ops, const AngularQuadrature& quad,
                            const BoundaryData& bc, const Vec& source, const Vec& phi_prev,
                            const LowRankParams& params, SubsampleRng& rng) {
  if (params.p < 1 || params.q < params.p) throw std::invalid_argument("low_rank_si: need 1 <= p <= q");
  const int n_omega = quad.size(), n = ops.space.size();
  Vec rhs_core = rhs_core_of(ops, phi_prev, source);
  LowRankBasis basis(ops, quad, bc, rhs_core);
  std::vector<char> sampled(n_omega, 0);
  InnerLoopResult out;
  Vec phi_old = phi_prev;
  std::vector<int> all(n_omega);
  std::iota(all.begin(), all.end(), 0);
  std::vector<int> next = rng.sample_without_replacement(all, std::min(params.p, n_omega));
  while (true) {
    ++out.iterations;
    const int p_now = static_cast<int>(next.size());
    Mat snaps(n, p_now);
    for (int i = 0; i < p_now; ++i) {
      const int j = next[i];
      Vec psi = sweep(ops, quad, j, with_bc(rhs_core, bc, j));
      std::copy(psi.begin(), psi.end(), snaps.col(i));
      sampled[j] = 1;
      out.sampled_order.push_back(j);
    }
    bool reorth = basis.mgs_ro_update(snaps, next, params.eps_mgs);
    basis.update_projections(reorth);
    if (reorth) ++out.reorthogonalizations;
    const bool any_unsampled = std::any_of(sampled.begin(), sampled.end(), [](char s) { return !s; });
    if (!any_unsampled) {
      out.exhausted_all_angles = true;
      out.coefficients = build_full_coefficients(basis, sampled, nullptr);
      out.phi_star = phi_from(basis, out.coefficients, quad.weights);
      break;
    }
    SubsampleOutcome sub = greedy_subsample(basis, sampled, params.p, params.q, rng);
    next = sub.selected;
    if (sub.max_residual < params.eps_res) {
      Mat c = build_full_coefficients(basis, sampled, &sub);
      Vec phi = phi_from(basis, c, quad.weights);
      Vec d(n);
      for (int i = 0; i < n; ++i) d[i] = phi[i] - phi_old[i];
      if (norm2(d) <= params.eps_diff) {
        std::vector<int> unsampled;
        for (int j = 0; j < n_omega; ++j)
          if (!sampled[j]) unsampled.push_back(j);
        std::vector<double> norms = batched_residual_norms(basis, unsampled, c);
        std::vector<std::pair<double, int>> outstanding;
        for (size_t i = 0; i < unsampled.size(); ++i)
          if (norms[i] >= params.eps_res) outstanding.push_back({norms[i], unsampled[i]});
        if (outstanding.empty()) {
          out.phi_star = std::move(phi);
          out.coefficients = std::move(c);
          break;
        }
        std::sort(outstanding.begin(), outstanding.end(), [](const auto& a, const auto& b) {
          if (a.first != b.first) return a.first > b.first;
          return a.second < b.second;
        });
        next.clear();
        for (const auto& e : outstanding) next.push_back(e.second);
        ++out.verification_rejections;
      }
      phi_old = std::move(phi);
    }
  }
  out.rank = basis.rank();
  out.sampled_count = basis.snapshot_count();
  out.basis = basis.basis();
  return out;
}

// proj/src/low_rank.cpp:436-492
SolveReport solve_low_rank(const DiscreteOperators& ops, const AngularQuadrature& quad,
                           const BoundaryData& bc, const Vec& source, const DiffusionSystem* dsa,
                           const LowRankOptions& opts) {
  if (opts.use_dsa && dsa == nullptr)
    throw std::invalid_argument("solve_low_rank: DSA requested but no diffusion system");
  const int n = ops.space.size(), n_omega = quad.size();
  SolveReport report;
  report.method = "lowrank";
  SubsampleRng rng(opts.seed);
  auto t0 = std::chrono::steady_clock::now();
  Vec phi(n, 0.0);
  InnerLoopResult inner;
  int final_rank = 0;
  for (int it = 1; it <= opts.max_iterations; ++it) {
    inner = low_rank_si(ops, quad, bc, source, phi, opts.inner, rng);
    Vec sv = svd_values(inner.coefficients);
    const int rp = truncation_rank(sv, opts.inner.eps_svd);
    Vec d(n);
    for (int i = 0; i < n; ++i) d[i] = inner.phi_star[i] - phi[i];
    OuterRecord rec;
    rec.diff_two_norm = norm2(d);
    rec.diff_inf_norm = norm_inf(d);
    rec.rank = rp;
    rec.oversampling = rp > 0 ? static_cast<double>(inner.rank - rp) / rp : 0.0;
    rec.inner_iterations = inner.iterations;
    rec.sampled_count = inner.sampled_count;
    rec.fullrank_fallback = inner.exhausted_all_angles;
    report.history.push_back(rec);
    report.sampled_log.push_back(inner.sampled_order);
    report.iterations = it;
    final_rank = rp;
    if (rec.diff_inf_norm <= opts.eps_si_sa) {
      report.converged = true;
      phi = inner.phi_star;
      break;
    }
    if (opts.use_dsa) {
      Vec delta = dsa->correct(inner.phi_star, phi);
      for (int i = 0; i < n; ++i) phi[i] = inner.phi_star[i] + delta[i];
    } else {
      phi = inner.phi_star;
    }
  }
  if (!report.converged) phi = inner.phi_star;
  report.solve_seconds =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  report.phi = phi;
  report.psi_dofs = static_cast<long long>(final_rank) * (n + n_omega);
  if (opts.build_factors) {
    report.has_factors = true;
    report.factors = truncate_factors(inner.coefficients, inner.basis, opts.inner.eps_svd);
  }
  return report;
}

// proj/src/report.cpp:47-58
double psi_difference(const Mat& psi_full, const LowRankFactors& f) {
  double acc = 0.0;
  const int r = f.rank();
  for (int j = 0; j < psi_full.cols; ++j)
    for (int i = 0; i < psi_full.rows; ++i) {
      double rec = 0.0;
      for (int k = 0; k < r; ++k) rec += f.X(i, k) * (f.S[k] * f.V(j, k));
      const double d = psi_full(i, j) - rec;
      acc += d * d;
    }
  return std::sqrt(acc);
}

}  // namespace oracle
