// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp header).
// Restates proj/src/quadrature.cpp, proj/src/dg_space.cpp,
// proj/src/operators.cpp, proj/src/sweep.cpp and the Eigen kernels they use.
#include <algorithm>
#include <cmath>
#include <map>

#include "oracle.hpp"

namespace oracle {

// ------------------------------------------------------------------ CSR
Csr csr_from_triplets(int n, const std::vector<Triplet>& t) {
  // Eigen::SparseMatrix::setFromTriplets: duplicates are summed in the order
  // the triplets were appended; inner indices sorted.
  std::vector<std::vector<std::pair<int, double>>> rows(n);
  for (const Triplet& e : t) rows[e.r].push_back({e.c, e.v});
  Csr m;
  m.n = n;
  m.rowptr.assign(n + 1, 0);
  for (int i = 0; i < n; ++i) {
    auto& r = rows[i];
    std::stable_sort(r.begin(), r.end(),
                     [](const auto& a, const auto& b) { return a.first < b.first; });
    std::vector<std::pair<int, double>> merged;
    for (auto& e : r) {
      if (!merged.empty() && merged.back().first == e.first)
        merged.back().second += e.second;
      else
        merged.push_back(e);
    }
    for (auto& e : merged) {
      m.colidx.push_back(e.first);
      m.val.push_back(e.second);
    }
    m.rowptr[i + 1] = static_cast<int>(m.colidx.size());
  }
  return m;
}

Csr csr_add(const Csr& a, const Csr& b) {
  Csr m;
  m.n = a.n;
  m.rowptr.assign(a.n + 1, 0);
  for (int i = 0; i < a.n; ++i) {
    int p = a.rowptr[i], pe = a.rowptr[i + 1], q = b.rowptr[i], qe = b.rowptr[i + 1];
    while (p < pe || q < qe) {
      if (q >= qe || (p < pe && a.colidx[p] < b.colidx[q])) {
        m.colidx.push_back(a.colidx[p]);
        m.val.push_back(a.val[p++]);
      } else if (p >= pe || b.colidx[q] < a.colidx[p]) {
        m.colidx.push_back(b.colidx[q]);
        m.val.push_back(b.val[q++]);
      } else {
        m.colidx.push_back(a.colidx[p]);
        m.val.push_back(a.val[p++] + b.val[q++]);
      }
    }
    m.rowptr[i + 1] = static_cast<int>(m.colidx.size());
  }
  return m;
}

Vec Csr::mul(const Vec& x) const {
  Vec y(n);
  for (int i = 0; i < n; ++i) {
    double tmp = 0.0;
    for (int k = rowptr[i]; k < rowptr[i + 1]; ++k) tmp += val[k] * x[colidx[k]];
    y[i] = tmp;
  }
  return y;
}

Vec Csr::tmul(const Vec& x) const {
  Vec y(n, 0.0);
  for (int i = 0; i < n; ++i)
    for (int k = rowptr[i]; k < rowptr[i + 1]; ++k) y[colidx[k]] += val[k] * x[i];
  return y;
}

Mat Csr::mul(const Mat& x) const {
  Mat y(n, x.cols);
  for (int c = 0; c < x.cols; ++c) {
    const double* xc = x.col(c);
    double* yc = y.col(c);
    for (int i = 0; i < n; ++i) {
      double tmp = 0.0;
      for (int k = rowptr[i]; k < rowptr[i + 1]; ++k) tmp += val[k] * xc[colidx[k]];
      yc[i] = tmp;
    }
  }
  return y;
}

Mat Csr::tmul(const Mat& x) const {
  Mat y(n, x.cols);
  for (int c = 0; c < x.cols; ++c) {
    const double* xc = x.col(c);
    double* yc = y.col(c);
    for (int i = 0; i < n; ++i)
      for (int k = rowptr[i]; k < rowptr[i + 1]; ++k) yc[colidx[k]] += val[k] * xc[i];
  }
  return y;
}

double Csr::at(int i, int j) const {
  for (int k = rowptr[i]; k < rowptr[i + 1]; ++k)
    if (colidx[k] == j) return val[k];
  return 0.0;
}

// ------------------------------------------------------------------ quadrature
// proj/src/quadrature.cpp:8-17
double legendre_value(int n, double x) {
  if (n == 0) return 1.0;
  double pm1 = 1.0, p = x;
  for (int k = 2; k <= n; ++k) {
    double pk = ((2.0 * k - 1.0) * x * p - (k - 1.0) * pm1) / k;
    pm1 = p;
    p = pk;
  }
  return p;
}

// proj/src/quadrature.cpp:19-27
double legendre_derivative(int n, double x) {
  if (n == 0) return 0.0;
  if (std::abs(1.0 - x * x) < 1e-14) {
    double sign = (x > 0.0 || n % 2 == 1) ? 1.0 : -1.0;
    return sign * 0.5 * n * (n + 1.0);
  }
  return n * (legendre_value(n - 1, x) - x * legendre_value(n, x)) / (1.0 - x * x);
}

// proj/src/quadrature.cpp:29-54 (Newton roots, mirrored nodes)
GaussLegendre gauss_legendre(int n) {
  if (n < 1) throw std::invalid_argument("gauss_legendre: need at least one node");
  GaussLegendre rule;
  rule.nodes.assign(n, 0.0);
  rule.weights.assign(n, 0.0);
  const int half = (n + 1) / 2;
  for (int i = 0; i < half; ++i) {
    double x = std::cos(M_PI * (i + 0.75) / (n + 0.5));
    for (int it = 0; it < 100; ++it) {
      double p = legendre_value(n, x);
      double dp = legendre_derivative(n, x);
      double dx = p / dp;
      x -= dx;
      if (std::abs(p) < 1e-15 && std::abs(dx) < 1e-15) break;
    }
    double dp = legendre_derivative(n, x);
    double w = 2.0 / ((1.0 - x * x) * dp * dp);
    rule.nodes[n - 1 - i] = x;
    rule.nodes[i] = -x;
    rule.weights[n - 1 - i] = w;
    rule.weights[i] = w;
  }
  if (n % 2 == 1) rule.nodes[half - 1] = 0.0;
  return rule;
}

// proj/src/quadrature.cpp:56-84 (azimuth-major j = j1 * n_omega_z + j2)
AngularQuadrature build_cl_quadrature(int n_theta, int n_omega_z) {
  if (n_theta < 1 || n_omega_z < 1)
    throw std::invalid_argument("build_cl_quadrature: node counts must be positive");
  GaussLegendre gl = gauss_legendre(n_omega_z);
  AngularQuadrature quad;
  quad.n_theta = n_theta;
  quad.n_omega_z = n_omega_z;
  const int n = n_theta * n_omega_z;
  quad.dirs.assign(3 * static_cast<size_t>(n), 0.0);
  quad.weights.assign(n, 0.0);
  const double w_theta = 1.0 / n_theta;
  for (int j1 = 0; j1 < n_theta; ++j1) {
    double theta = (2.0 * j1 + 1.0) * M_PI / n_theta;
    double c = std::cos(theta), s = std::sin(theta);
    for (int j2 = 0; j2 < n_omega_z; ++j2) {
      double z = gl.nodes[j2];
      double rho = std::sqrt(1.0 - z * z);
      int j = j1 * n_omega_z + j2;
      quad.dirs[3 * j] = c * rho;
      quad.dirs[3 * j + 1] = s * rho;
      quad.dirs[3 * j + 2] = z;
      quad.weights[j] = w_theta * (0.5 * gl.weights[j2]);
    }
  }
  return quad;
}

// ------------------------------------------------------------------ mesh / DG
// proj/src/dg_space.cpp:11-53
SpatialMesh make_mesh(double x_min, double x_max, double y_min, double y_max, int nx, int ny) {
  if (!(x_min < x_max) || !(y_min < y_max)) throw std::invalid_argument("make_mesh: empty domain");
  if (nx < 1 || ny < 1) throw std::invalid_argument("make_mesh: cell counts must be positive");
  SpatialMesh m;
  m.x_min = x_min;
  m.x_max = x_max;
  m.y_min = y_min;
  m.y_max = y_max;
  m.nx = nx;
  m.ny = ny;
  return m;
}

double DGSpace::basis_1d_x(int m, int a, double x) const {
  double h = mesh.dx();
  double xi = 2.0 * (x - mesh.x_center(a)) / h;
  return std::sqrt((2.0 * m + 1.0) / h) * legendre_value(m, xi);
}
double DGSpace::basis_1d_y(int m, int b, double y) const {
  double h = mesh.dy();
  double eta = 2.0 * (y - mesh.y_center(b)) / h;
  return std::sqrt((2.0 * m + 1.0) / h) * legendre_value(m, eta);
}
double DGSpace::basis_value(int cell, int tensor, double x, double y) const {
  int a = cell % mesh.nx, b = cell / mesh.nx;
  int mx = tensor % (degree + 1), my = tensor / (degree + 1);
  return basis_1d_x(mx, a, x) * basis_1d_y(my, b, y);
}
double DGSpace::cell_mean(const Vec& coeffs, int cell) const {
  return coeffs[cell * dofs_per_cell()] / std::sqrt(mesh.dx() * mesh.dy());
}
DGSpace build_dg_space(const SpatialMesh& mesh, int degree) {
  if (degree < 0) throw std::invalid_argument("build_dg_space: negative degree");
  DGSpace s;
  s.mesh = mesh;
  s.degree = degree;
  return s;
}

// ------------------------------------------------------------------ operators
namespace {

// proj/src/operators.cpp:13-21
Mat derivative_matrix_1d(int degree, double h) {
  int n = degree + 1;
  Mat d(n, n);
  for (int m = 0; m < n; ++m)
    for (int l = 0; l < n; ++l)
      if (m > l && (m - l) % 2 == 1) d(m, l) = 2.0 * std::sqrt((2.0 * m + 1.0) * (2.0 * l + 1.0)) / h;
  return d;
}
// proj/src/operators.cpp:24-35
Vec trace_right_1d(int degree, double h) {
  Vec t(degree + 1);
  for (int m = 0; m <= degree; ++m) t[m] = std::sqrt((2.0 * m + 1.0) / h);
  return t;
}
Vec trace_left_1d(int degree, double h) {
  Vec t = trace_right_1d(degree, h);
  for (int m = 0; m <= degree; ++m)
    if (m % 2 == 1) t[m] = -t[m];
  return t;
}
struct Blocks1d {
  Mat a_minus, a_plus, b_minus, b_plus;
};
// proj/src/operators.cpp:47-57
Blocks1d streaming_blocks_1d(int degree, double h) {
  Mat v = derivative_matrix_1d(degree, h);
  Vec tr = trace_right_1d(degree, h), tl = trace_left_1d(degree, h);
  int n = degree + 1;
  Blocks1d b{Mat(n, n), Mat(n, n), Mat(n, n), Mat(n, n)};
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      b.a_minus(i, j) = -v(i, j) + tr[i] * tr[j];
      b.a_plus(i, j) = -v(i, j) - tl[i] * tl[j];
      b.b_minus(i, j) = -tl[i] * tr[j];
      b.b_plus(i, j) = tr[i] * tl[j];
    }
  return b;
}
// proj/src/operators.cpp:61-79
Mat tensor_x(const Mat& bx, int degree) {
  int n = degree + 1, s = n * n;
  Mat out(s, s);
  for (int my = 0; my < n; ++my)
    for (int mx = 0; mx < n; ++mx)
      for (int lx = 0; lx < n; ++lx) out(my * n + mx, my * n + lx) = bx(mx, lx);
  return out;
}
Mat tensor_y(const Mat& by, int degree) {
  int n = degree + 1, s = n * n;
  Mat out(s, s);
  for (int mx = 0; mx < n; ++mx)
    for (int my = 0; my < n; ++my)
      for (int ly = 0; ly < n; ++ly) out(my * n + mx, ly * n + mx) = by(my, ly);
  return out;
}
// proj/src/operators.cpp:81-85 (skip exact zeros, row-major block order)
void append_block(std::vector<Triplet>& t, int r0, int c0, const Mat& blk) {
  for (int i = 0; i < blk.rows; ++i)
    for (int j = 0; j < blk.cols; ++j)
      if (blk(i, j) != 0.0) t.push_back({r0 + i, c0 + j, blk(i, j)});
}

}  // namespace

// proj/src/operators.cpp:89-189
DiscreteOperators assemble_operators(const DGSpace& space, const Field& sigma_s_field,
                                     const Field& sigma_a_field) {
  const SpatialMesh& mesh = space.mesh;
  const int k = space.degree, n1 = k + 1, s = space.dofs_per_cell(), n = space.size();
  const double dx = mesh.dx(), dy = mesh.dy();
  DiscreteOperators ops;
  ops.space = space;
  Blocks1d bx = streaming_blocks_1d(k, dx), by = streaming_blocks_1d(k, dy);
  ops.ax_minus = tensor_x(bx.a_minus, k);
  ops.ax_plus = tensor_x(bx.a_plus, k);
  ops.bx_minus = tensor_x(bx.b_minus, k);
  ops.bx_plus = tensor_x(bx.b_plus, k);
  ops.ay_minus = tensor_y(by.a_minus, k);
  ops.ay_plus = tensor_y(by.a_plus, k);
  ops.by_minus = tensor_y(by.b_minus, k);
  ops.by_plus = tensor_y(by.b_plus, k);

  std::vector<Triplet> txm, txp, tym, typ;
  for (int b = 0; b < mesh.ny; ++b)
    for (int a = 0; a < mesh.nx; ++a) {
      int c = mesh.cell_index(a, b), r0 = c * s;
      append_block(txm, r0, r0, ops.ax_minus);
      append_block(txp, r0, r0, ops.ax_plus);
      append_block(tym, r0, r0, ops.ay_minus);
      append_block(typ, r0, r0, ops.ay_plus);
      if (a > 0) append_block(txm, r0, mesh.cell_index(a - 1, b) * s, ops.bx_minus);
      if (a + 1 < mesh.nx) append_block(txp, r0, mesh.cell_index(a + 1, b) * s, ops.bx_plus);
      if (b > 0) append_block(tym, r0, mesh.cell_index(a, b - 1) * s, ops.by_minus);
      if (b + 1 < mesh.ny) append_block(typ, r0, mesh.cell_index(a, b + 1) * s, ops.by_plus);
    }
  ops.d_x_minus = csr_from_triplets(n, txm);
  ops.d_x_plus = csr_from_triplets(n, txp);
  ops.d_y_minus = csr_from_triplets(n, tym);
  ops.d_y_plus = csr_from_triplets(n, typ);

  const int nq = k + 2;
  GaussLegendre gl = gauss_legendre(nq);
  Mat bxv(n1, nq), byv(n1, nq);
  for (int m = 0; m < n1; ++m)
    for (int g = 0; g < nq; ++g) {
      bxv(m, g) = std::sqrt((2.0 * m + 1.0) / dx) * legendre_value(m, gl.nodes[g]);
      byv(m, g) = std::sqrt((2.0 * m + 1.0) / dy) * legendre_value(m, gl.nodes[g]);
    }
  std::vector<Triplet> ts, tt, ta;
  ops.sigma_t_blocks.resize(mesh.cell_count());
  Vec eta(s);
  for (int b = 0; b < mesh.ny; ++b)
    for (int a = 0; a < mesh.nx; ++a) {
      int c = mesh.cell_index(a, b);
      Mat bs(s, s), babs(s, s);
      for (int gy = 0; gy < nq; ++gy) {
        double y = mesh.y_center(b) + 0.5 * dy * gl.nodes[gy];
        for (int gx = 0; gx < nq; ++gx) {
          double x = mesh.x_center(a) + 0.5 * dx * gl.nodes[gx];
          double ss = sigma_s_field(x, y), sa = sigma_a_field(x, y);
          if (ss < 0.0 || sa < 0.0)
            throw std::invalid_argument("assemble_operators: negative cross section");
          double w = gl.weights[gx] * gl.weights[gy] * 0.25 * dx * dy;
          for (int my = 0; my < n1; ++my)
            for (int mx = 0; mx < n1; ++mx) eta[my * n1 + mx] = bxv(mx, gx) * byv(my, gy);
          // bs.noalias() += (w*ss) * (eta * eta^T)   (operators.cpp:170).
          // Eigen folds the scalar into the left factor of the outer
          // product: entry (i,j) += (alpha*eta_i) * eta_j.
          double ws = w * ss, wa = w * sa;
          for (int j = 0; j < s; ++j)
            for (int i = 0; i < s; ++i) {
              bs(i, j) += (ws * eta[i]) * eta[j];
              babs(i, j) += (wa * eta[i]) * eta[j];
            }
        }
      }
      int r0 = c * s;
      append_block(ts, r0, r0, bs);
      append_block(ta, r0, r0, babs);
      Mat bt(s, s);
      for (size_t i = 0; i < bt.a.size(); ++i) bt.a[i] = bs.a[i] + babs.a[i];
      append_block(tt, r0, r0, bt);
      ops.sigma_t_blocks[c] = bt;
    }
  ops.sigma_s = csr_from_triplets(n, ts);
  ops.sigma_t = csr_from_triplets(n, tt);
  ops.sigma_a = csr_from_triplets(n, ta);
  return ops;
}

// proj/src/operators.cpp:191-225
Vec project_source(const DGSpace& space, const Field& g) {
  const SpatialMesh& mesh = space.mesh;
  const int k = space.degree, n1 = k + 1, s = space.dofs_per_cell(), nq = k + 2;
  const double dx = mesh.dx(), dy = mesh.dy();
  GaussLegendre gl = gauss_legendre(nq);
  Mat bxv(n1, nq), byv(n1, nq);
  for (int m = 0; m < n1; ++m)
    for (int q = 0; q < nq; ++q) {
      bxv(m, q) = std::sqrt((2.0 * m + 1.0) / dx) * legendre_value(m, gl.nodes[q]);
      byv(m, q) = std::sqrt((2.0 * m + 1.0) / dy) * legendre_value(m, gl.nodes[q]);
    }
  Vec out(space.size(), 0.0);
  for (int b = 0; b < mesh.ny; ++b)
    for (int a = 0; a < mesh.nx; ++a) {
      int c = mesh.cell_index(a, b);
      for (int gy = 0; gy < nq; ++gy) {
        double y = mesh.y_center(b) + 0.5 * dy * gl.nodes[gy];
        for (int gx = 0; gx < nq; ++gx) {
          double x = mesh.x_center(a) + 0.5 * dx * gl.nodes[gx];
          double w = gl.weights[gx] * gl.weights[gy] * 0.25 * dx * dy * g(x, y);
          if (w == 0.0) continue;
          for (int my = 0; my < n1; ++my)
            for (int mx = 0; mx < n1; ++mx) out[c * s + my * n1 + mx] += w * bxv(mx, gx) * byv(my, gy);
        }
      }
    }
  return out;
}

// proj/src/operators.cpp:227-281
Vec boundary_vector(const DGSpace& space, const AngularQuadrature& quad, const Field& g,
                    int angle) {
  if (angle < 0 || angle >= quad.size())
    throw std::invalid_argument("boundary_vector: angle index out of range");
  const SpatialMesh& mesh = space.mesh;
  const int k = space.degree, n1 = k + 1, s = space.dofs_per_cell(), nq = k + 2;
  const double dx = mesh.dx(), dy = mesh.dy();
  const double omx = quad.omega_x(angle), omy = quad.omega_y(angle);
  GaussLegendre gl = gauss_legendre(nq);
  Vec trx_l = trace_left_1d(k, dx), trx_r = trace_right_1d(k, dx);
  Vec try_l = trace_left_1d(k, dy), try_r = trace_right_1d(k, dy);
  Vec out(space.size(), 0.0);
  auto add_x_edge = [&](int a, double x_edge, const Vec& trx, double coeff) {
    for (int b = 0; b < mesh.ny; ++b) {
      int c = mesh.cell_index(a, b);
      for (int q = 0; q < nq; ++q) {
        double y = mesh.y_center(b) + 0.5 * dy * gl.nodes[q];
        double w = coeff * gl.weights[q] * 0.5 * dy * g(x_edge, y);
        if (w == 0.0) continue;
        for (int my = 0; my < n1; ++my) {
          double byv = space.basis_1d_y(my, b, y);
          for (int mx = 0; mx < n1; ++mx) out[c * s + my * n1 + mx] += w * trx[mx] * byv;
        }
      }
    }
  };
  auto add_y_edge = [&](int b, double y_edge, const Vec& tryv, double coeff) {
    for (int a = 0; a < mesh.nx; ++a) {
      int c = mesh.cell_index(a, b);
      for (int q = 0; q < nq; ++q) {
        double x = mesh.x_center(a) + 0.5 * dx * gl.nodes[q];
        double w = coeff * gl.weights[q] * 0.5 * dx * g(x, y_edge);
        if (w == 0.0) continue;
        for (int mx = 0; mx < n1; ++mx) {
          double bxv = space.basis_1d_x(mx, a, x);
          for (int my = 0; my < n1; ++my) out[c * s + my * n1 + mx] += w * tryv[my] * bxv;
        }
      }
    }
  };
  if (omx > 0.0) add_x_edge(0, mesh.x_min, trx_l, omx);
  if (omx < 0.0) add_x_edge(mesh.nx - 1, mesh.x_max, trx_r, -omx);
  if (omy > 0.0) add_y_edge(0, mesh.y_min, try_l, omy);
  if (omy < 0.0) add_y_edge(mesh.ny - 1, mesh.y_max, try_r, -omy);
  return out;
}

// proj/src/operators.cpp:283-288
Vec StreamingOperator::apply(const Vec& v) const {
  Vec out = ops->sigma_t.mul(v);
  if (omega_x != 0.0) {
    Vec t = dx->mul(v);
    for (size_t i = 0; i < out.size(); ++i) out[i] += omega_x * t[i];
  }
  if (omega_y != 0.0) {
    Vec t = dy->mul(v);
    for (size_t i = 0; i < out.size(); ++i) out[i] += omega_y * t[i];
  }
  return out;
}

Mat StreamingOperator::materialize_dense() const {
  int n = ops->sigma_t.n;
  Mat m(n, n);
  auto add = [&](const Csr& a, double f) {
    for (int i = 0; i < n; ++i)
      for (int k = a.rowptr[i]; k < a.rowptr[i + 1]; ++k) m(i, a.colidx[k]) += f * a.val[k];
  };
  add(ops->sigma_t, 1.0);
  if (omega_x != 0.0) add(*dx, omega_x);
  if (omega_y != 0.0) add(*dy, omega_y);
  return m;
}

// proj/src/operators.cpp:297-308 (Omega >= 0 -> "minus" matrices)
StreamingOperator upwind_combination(const DiscreteOperators& ops, double omx, double omy) {
  StreamingOperator op;
  op.ops = &ops;
  op.omega_x = omx;
  op.omega_y = omy;
  op.dx = omx >= 0.0 ? &ops.d_x_minus : &ops.d_x_plus;
  op.dy = omy >= 0.0 ? &ops.d_y_minus : &ops.d_y_plus;
  return op;
}
StreamingOperator upwind_combination(const DiscreteOperators& ops, const AngularQuadrature& quad,
                                     int angle) {
  if (angle < 0 || angle >= quad.size())
    throw std::invalid_argument("upwind_combination: angle index out of range");
  return upwind_combination(ops, quad.omega_x(angle), quad.omega_y(angle));
}

// ------------------------------------------------------------------ dense LA
double dot(const double* a, const double* b, int n) {
  double s = 0.0;
  for (int i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}
double norm2(const Vec& v) { return std::sqrt(dot(v.data(), v.data(), static_cast<int>(v.size()))); }
double norm_inf(const Vec& v) {
  double m = 0.0;
  for (double x : v) m = std::max(m, std::abs(x));
  return m;
}

// Eigen::PartialPivLU unblocked kernel: first-max pivot, column scaled by
// division, rank-1 trailing update (Eigen/src/LU/PartialPivLU.h).
void LU::compute(const Mat& a) {
  lu = a;
  const int n = a.rows;
  perm.assign(n, 0);
  for (int k = 0; k < n; ++k) {
    int piv = k;
    double big = std::abs(lu(k, k));
    for (int i = k + 1; i < n; ++i)
      if (std::abs(lu(i, k)) > big) {
        big = std::abs(lu(i, k));
        piv = i;
      }
    perm[k] = piv;
    if (big != 0.0) {
      if (piv != k)
        for (int j = 0; j < n; ++j) std::swap(lu(k, j), lu(piv, j));
      const double d = lu(k, k);
      for (int i = k + 1; i < n; ++i) lu(i, k) /= d;
    }
    for (int j = k + 1; j < n; ++j) {
      const double u = lu(k, j);
      for (int i = k + 1; i < n; ++i) lu(i, j) -= lu(i, k) * u;
    }
  }
}

// Column-oriented unit-lower then upper substitution (Eigen
// triangular_solve_vector for ColMajor).
Vec LU::solve(const Vec& b) const {
  const int n = lu.rows;
  Vec x = b;
  for (int k = 0; k < n; ++k) std::swap(x[k], x[perm[k]]);
  for (int i = 0; i < n; ++i) {
    const double xi = x[i];
    for (int j = i + 1; j < n; ++j) x[j] -= xi * lu(j, i);
  }
  for (int i = n - 1; i >= 0; --i) {
    x[i] /= lu(i, i);
    const double xi = x[i];
    for (int j = 0; j < i; ++j) x[j] -= xi * lu(j, i);
  }
  return x;
}

double LU::min_abs_diag() const {
  double m = std::abs(lu(0, 0));
  for (int i = 1; i < lu.rows; ++i) m = std::min(m, std::abs(lu(i, i)));
  return m;
}

// Eigen HouseholderQR (makeHouseholder: beta = -sign(c0)*||x||).
void householder_qr(const Mat& a, Mat& thin_q, Mat& r) {
  const int m = a.rows, n = a.cols;
  Mat qr = a;
  Vec tau(n, 0.0);
  for (int k = 0; k < n && k < m; ++k) {
    double* x = qr.col(k) + k;
    const int len = m - k;
    double tail = 0.0;
    for (int i = 1; i < len; ++i) tail += x[i] * x[i];
    const double c0 = x[0];
    double beta, t;
    if (tail <= std::numeric_limits<double>::min()) {
      t = 0.0;
      beta = c0;
      for (int i = 1; i < len; ++i) x[i] = 0.0;
    } else {
      beta = std::sqrt(c0 * c0 + tail);
      if (c0 >= 0.0) beta = -beta;
      const double denom = c0 - beta;
      for (int i = 1; i < len; ++i) x[i] /= denom;
      t = (beta - c0) / beta;
    }
    tau[k] = t;
    x[0] = beta;
    // apply H = I - t v v^T (v = [1; x[1:]]) to the remaining columns
    for (int j = k + 1; j < n; ++j) {
      double* y = qr.col(j) + k;
      double w = y[0];
      for (int i = 1; i < len; ++i) w += x[i] * y[i];
      w *= t;
      y[0] -= w;
      for (int i = 1; i < len; ++i) y[i] -= w * x[i];
    }
  }
  const int kk = std::min(m, n);
  r = Mat(n, n);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i <= j && i < kk; ++i) r(i, j) = qr(i, j);
  thin_q = Mat(m, n);
  for (int j = 0; j < n && j < m; ++j) thin_q(j, j) = 1.0;
  for (int k = kk - 1; k >= 0; --k) {
    const double* v = qr.col(k) + k;
    const int len = m - k;
    for (int j = 0; j < n; ++j) {
      double* y = thin_q.col(j) + k;
      double w = y[0];
      for (int i = 1; i < len; ++i) w += v[i] * y[i];
      w *= tau[k];
      y[0] -= w;
      for (int i = 1; i < len; ++i) y[i] -= w * v[i];
    }
  }
}

namespace {
// One-sided (Hestenes) Jacobi on the columns of w (m x n, m >= n): w <- w*J,
// j accumulates J.  Returns nothing; columns of w end mutually orthogonal.
void jacobi_columns(Mat& w, Mat* j) {
  const int m = w.rows, n = w.cols;
  for (int sweep = 0; sweep < 60; ++sweep) {
    bool rotated = false;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        double* wp = w.col(p);
        double* wq = w.col(q);
        double alpha = 0, beta = 0, gamma = 0;
        for (int i = 0; i < m; ++i) {
          alpha += wp[i] * wp[i];
          beta += wq[i] * wq[i];
          gamma += wp[i] * wq[i];
        }
        if (gamma == 0.0 || std::abs(gamma) <= 1e-15 * std::sqrt(alpha * beta)) continue;
        rotated = true;
        const double zeta = (beta - alpha) / (2.0 * gamma);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / std::sqrt(1.0 + t * t), s = c * t;
        for (int i = 0; i < m; ++i) {
          const double a = wp[i], b = wq[i];
          wp[i] = c * a - s * b;
          wq[i] = s * a + c * b;
        }
        if (j) {
          double* jp = j->col(p);
          double* jq = j->col(q);
          for (int i = 0; i < j->rows; ++i) {
            const double a = jp[i], b = jq[i];
            jp[i] = c * a - s * b;
            jq[i] = s * a + c * b;
          }
        }
      }
    if (!rotated) break;
  }
}
}  // namespace

void svd_thin(const Mat& a, Mat* u, Vec& s, Mat* v) {
  // For m >= n Jacobi on A: A J = U S.  For m < n Jacobi on A^T: A^T J = V S,
  // so A = J S V^T.  A Householder QR preconditions the tall side.
  const bool tall = a.rows >= a.cols;
  Mat t;
  if (tall) {
    t = a;
  } else {
    t = Mat(a.cols, a.rows);
    for (int i = 0; i < a.rows; ++i)
      for (int j = 0; j < a.cols; ++j) t(j, i) = a(i, j);
  }
  const int m = t.rows, n = t.cols;
  Mat q, r;
  householder_qr(t, q, r);  // t = q r, r is n x n
  Mat w = r;
  Mat jm = Mat::identity(n);
  jacobi_columns(w, &jm);
  std::vector<double> sv(n);
  for (int k = 0; k < n; ++k) sv[k] = std::sqrt(dot(w.col(k), w.col(k), n));
  std::vector<int> order(n);
  for (int k = 0; k < n; ++k) order[k] = k;
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return sv[x] > sv[y]; });
  s.assign(n, 0.0);
  Mat left(m, n), right(n, n);  // t = left * diag(s) * right^T
  for (int kk = 0; kk < n; ++kk) {
    const int k = order[kk];
    s[kk] = sv[k];
    Vec uk(n, 0.0);
    if (sv[k] > 0.0)
      for (int i = 0; i < n; ++i) uk[i] = w(i, k) / sv[k];
    else
      uk[kk] = 1.0;
    // left column = q * uk
    for (int i = 0; i < m; ++i) {
      double acc = 0.0;
      for (int l = 0; l < n; ++l) acc += q(i, l) * uk[l];
      left(i, kk) = acc;
    }
    for (int i = 0; i < n; ++i) right(i, kk) = jm(i, k);
  }
  if (tall) {
    if (u) *u = left;
    if (v) *v = right;
  } else {
    if (u) *u = right;
    if (v) *v = left;
  }
}

Vec svd_values(const Mat& a) {
  Vec s;
  svd_thin(a, nullptr, s, nullptr);
  return s;
}

// ------------------------------------------------------------------ sweep
// proj/src/sweep.cpp:9-57: one upwind block Gauss-Seidel pass, b outer,
// a inner, per-cell partial-pivot LU with the singular-block test.
Vec sweep(const DiscreteOperators& ops, double omx, double omy, const Vec& rhs) {
  const SpatialMesh& mesh = ops.space.mesh;
  const int s = ops.space.dofs_per_cell();
  if (static_cast<int>(rhs.size()) != ops.space.size())
    throw std::invalid_argument("sweep: rhs size mismatch");
  const bool x_up = omx >= 0.0, y_up = omy >= 0.0;
  const Mat& ax = x_up ? ops.ax_minus : ops.ax_plus;
  const Mat& ay = y_up ? ops.ay_minus : ops.ay_plus;
  const Mat& bx = x_up ? ops.bx_minus : ops.bx_plus;
  const Mat& by = y_up ? ops.by_minus : ops.by_plus;
  const int x_step = x_up ? 1 : -1, y_step = y_up ? 1 : -1;
  Vec psi(rhs.size(), 0.0);
  Mat block(s, s);
  Vec local(s);
  LU lu;
  int b = y_up ? 0 : mesh.ny - 1;
  for (int jb = 0; jb < mesh.ny; ++jb, b += y_step) {
    int a = x_up ? 0 : mesh.nx - 1;
    for (int ja = 0; ja < mesh.nx; ++ja, a += x_step) {
      const int c = mesh.cell_index(a, b);
      for (int i = 0; i < s; ++i) local[i] = rhs[c * s + i];
      const int an = a - x_step, bn = b - y_step;
      if (an >= 0 && an < mesh.nx) {
        const double* up = psi.data() + mesh.cell_index(an, b) * s;
        for (int i = 0; i < s; ++i) {
          double t = 0.0;
          for (int j = 0; j < s; ++j) t += bx(i, j) * up[j];
          local[i] -= omx * t;
        }
      }
      if (bn >= 0 && bn < mesh.ny) {
        const double* up = psi.data() + mesh.cell_index(a, bn) * s;
        for (int i = 0; i < s; ++i) {
          double t = 0.0;
          for (int j = 0; j < s; ++j) t += by(i, j) * up[j];
          local[i] -= omy * t;
        }
      }
      const Mat& st = ops.sigma_t_blocks[c];
      double amax = 0.0;
      for (int j = 0; j < s; ++j)
        for (int i = 0; i < s; ++i) {
          block(i, j) = omx * ax(i, j) + omy * ay(i, j) + st(i, j);
          amax = std::max(amax, std::abs(block(i, j)));
        }
      lu.compute(block);
      if (!(lu.min_abs_diag() > 1e-14 * amax)) throw std::runtime_error("sweep: singular local block");
      Vec sol = lu.solve(local);
      for (int i = 0; i < s; ++i) psi[c * s + i] = sol[i];
    }
  }
  return psi;
}

Vec sweep(const DiscreteOperators& ops, const AngularQuadrature& quad, int angle, const Vec& rhs) {
  if (angle < 0 || angle >= quad.size()) throw std::invalid_argument("sweep: angle index out of range");
  return sweep(ops, quad.omega_x(angle), quad.omega_y(angle), rhs);
}

}  // namespace oracle
