// Host assembly for DG degree K != 1 (the GPU sweep/apply path for any K;
// the solvers and the DSA are K = 1).  Same arithmetic, expression by
// expression, as the reference's general-K code:
//   streaming blocks   proj/src/operators.cpp:13-79, 101-112
//   cross sections     proj/src/operators.cpp:137-181 ((K+2)^2 Gauss points)
//   source projection  proj/src/operators.cpp:191-225
//   boundary vectors   proj/src/operators.cpp:227-281, full_rank.cpp:11-39
// Blocks are stored s x s column-major (s = (K+1)^2), like the K = 1 arrays.
#include <algorithm>
#include <chrono>
#include <cmath>

#include "host.hpp"

namespace rtlr {
namespace cuda {

namespace {

using Mat = std::vector<double>;  // n x n column-major

// operators.cpp:13-21
Mat derivative_matrix_1d(int degree, double h) {
  const int n = degree + 1;
  Mat d(static_cast<size_t>(n) * n, 0.0);
  for (int m = 0; m < n; ++m)
    for (int l = 0; l < n; ++l)
      if (m > l && (m - l) % 2 == 1) d[m + l * n] = 2.0 * std::sqrt((2.0 * m + 1.0) * (2.0 * l + 1.0)) / h;
  return d;
}

// operators.cpp:24-35
std::vector<double> trace_right_1d(int degree, double h) {
  std::vector<double> t(degree + 1);
  for (int m = 0; m <= degree; ++m) t[m] = std::sqrt((2.0 * m + 1.0) / h);
  return t;
}
std::vector<double> trace_left_1d(int degree, double h) {
  std::vector<double> t = trace_right_1d(degree, h);
  for (int m = 0; m <= degree; ++m)
    if (m % 2 == 1) t[m] = -t[m];
  return t;
}

// operators.cpp:47-57: a- = -V + trR trR^T, a+ = -V - trL trL^T,
// b- = -trL trR^T, b+ = trR trL^T
void streaming_blocks_1d(int degree, double h, Mat& am, Mat& ap, Mat& bm, Mat& bp) {
  const int n = degree + 1;
  const Mat v = derivative_matrix_1d(degree, h);
  const std::vector<double> tr = trace_right_1d(degree, h), tl = trace_left_1d(degree, h);
  am.assign(static_cast<size_t>(n) * n, 0.0);
  ap = am;
  bm = am;
  bp = am;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      am[i + j * n] = -v[i + j * n] + tr[i] * tr[j];
      ap[i + j * n] = -v[i + j * n] - tl[i] * tl[j];
      bm[i + j * n] = -tl[i] * tr[j];
      bp[i + j * n] = tr[i] * tl[j];
    }
}

// operators.cpp:61-79: the 1D block paired with the identity in the other coordinate
Mat tensor_x(const Mat& bx, int degree) {
  const int n = degree + 1, s = n * n;
  Mat out(static_cast<size_t>(s) * s, 0.0);
  for (int my = 0; my < n; ++my)
    for (int mx = 0; mx < n; ++mx)
      for (int lx = 0; lx < n; ++lx) out[(my * n + mx) + static_cast<size_t>(my * n + lx) * s] = bx[mx + lx * n];
  return out;
}
Mat tensor_y(const Mat& by, int degree) {
  const int n = degree + 1, s = n * n;
  Mat out(static_cast<size_t>(s) * s, 0.0);
  for (int mx = 0; mx < n; ++mx)
    for (int my = 0; my < n; ++my)
      for (int ly = 0; ly < n; ++ly) out[(my * n + mx) + static_cast<size_t>(ly * n + mx) * s] = by[my + ly * n];
  return out;
}

}  // namespace

void boundary_vector_general(const HostProblem& hp, const Field& g, int angle, double* out) {
  // operators.cpp:227-281 for any degree
  if (angle < 0 || angle >= hp.n_omega) throw std::invalid_argument("boundary_vector: angle index out of range");
  const ProblemConfig& cfg = hp.cfg;
  const int k = hp.degree, n1 = k + 1, s = hp.spc, nq = k + 2;
  const double dx = hp.dx, dy = hp.dy;
  const double omx = hp.dirs[3 * angle], omy = hp.dirs[3 * angle + 1];
  std::vector<double> gn, gw;
  gauss_legendre(nq, gn, gw);
  const std::vector<double> trx_l = trace_left_1d(k, dx), trx_r = trace_right_1d(k, dx);
  const std::vector<double> try_l = trace_left_1d(k, dy), try_r = trace_right_1d(k, dy);
  std::fill(out, out + hp.ndof, 0.0);
  auto x_center = [&](int a) { return cfg.x_min + (a + 0.5) * ((cfg.x_max - cfg.x_min) / cfg.nx); };
  auto y_center = [&](int b) { return cfg.y_min + (b + 0.5) * ((cfg.y_max - cfg.y_min) / cfg.ny); };
  auto basis_x = [&](int m, int a, double x) {
    const double xi = 2.0 * (x - x_center(a)) / dx;
    return std::sqrt((2.0 * m + 1.0) / dx) * legendre_value(m, xi);
  };
  auto basis_y = [&](int m, int b, double y) {
    const double eta = 2.0 * (y - y_center(b)) / dy;
    return std::sqrt((2.0 * m + 1.0) / dy) * legendre_value(m, eta);
  };
  auto add_x_edge = [&](int a, double x_edge, const std::vector<double>& trx, double coeff) {
    for (int b = 0; b < hp.ny; ++b) {
      const int c = b * hp.nx + a;
      for (int q = 0; q < nq; ++q) {
        const double y = y_center(b) + 0.5 * dy * gn[q];
        const double w = coeff * gw[q] * 0.5 * dy * g(x_edge, y);
        if (w == 0.0) continue;
        for (int my = 0; my < n1; ++my) {
          const double by = basis_y(my, b, y);
          for (int mx = 0; mx < n1; ++mx) out[static_cast<size_t>(c) * s + my * n1 + mx] += w * trx[mx] * by;
        }
      }
    }
  };
  auto add_y_edge = [&](int b, double y_edge, const std::vector<double>& tryv, double coeff) {
    for (int a = 0; a < hp.nx; ++a) {
      const int c = b * hp.nx + a;
      for (int q = 0; q < nq; ++q) {
        const double x = x_center(a) + 0.5 * dx * gn[q];
        const double w = coeff * gw[q] * 0.5 * dx * g(x, y_edge);
        if (w == 0.0) continue;
        for (int mx = 0; mx < n1; ++mx) {
          const double bx = basis_x(mx, a, x);
          for (int my = 0; my < n1; ++my) out[static_cast<size_t>(c) * s + my * n1 + mx] += w * tryv[my] * bx;
        }
      }
    }
  };
  if (omx > 0.0) add_x_edge(0, cfg.x_min, trx_l, omx);
  if (omx < 0.0) add_x_edge(hp.nx - 1, cfg.x_max, trx_r, -omx);
  if (omy > 0.0) add_y_edge(0, cfg.y_min, try_l, omy);
  if (omy < 0.0) add_y_edge(hp.ny - 1, cfg.y_max, try_r, -omy);
}

void assemble_general(const ProblemConfig& cfg, HostProblem& hp) {
  const auto t0 = std::chrono::steady_clock::now();
  validate_config(cfg);
  if (cfg.degree < 0 || cfg.degree > kMaxDegree)
    throw std::invalid_argument("rtlr::cuda: DG degree K must be in 0.." + std::to_string(kMaxDegree) +
                                " on the GPU path");
  const int k = cfg.degree, n1 = k + 1, s = n1 * n1, nq = k + 2;
  hp.cfg = cfg;
  hp.degree = k;
  hp.spc = s;
  hp.nx = cfg.nx;
  hp.ny = cfg.ny;
  hp.ncell = cfg.nx * cfg.ny;
  hp.ndof = s * hp.ncell;
  hp.dx = (cfg.x_max - cfg.x_min) / cfg.nx;  // SpatialMesh::dx (dg_space.hpp:19)
  hp.dy = (cfg.y_max - cfg.y_min) / cfg.ny;
  build_cl_quadrature(cfg.n_theta, cfg.n_omega_z, hp.dirs, hp.weights);
  hp.n_omega = cfg.n_theta * cfg.n_omega_z;
  const double dx = hp.dx, dy = hp.dy;
  auto x_center = [&](int a) { return cfg.x_min + (a + 0.5) * ((cfg.x_max - cfg.x_min) / cfg.nx); };
  auto y_center = [&](int b) { return cfg.y_min + (b + 0.5) * ((cfg.y_max - cfg.y_min) / cfg.ny); };

  // streaming blocks: ax-, ax+, ay-, ay+, bx-, bx+, by-, by+
  Mat amx, apx, bmx, bpx, amy, apy, bmy, bpy;
  streaming_blocks_1d(k, dx, amx, apx, bmx, bpx);
  streaming_blocks_1d(k, dy, amy, apy, bmy, bpy);
  const size_t ss = static_cast<size_t>(s) * s;
  hp.kblocks.assign(8 * ss, 0.0);
  const Mat blocks[8] = {tensor_x(amx, k), tensor_x(apx, k), tensor_y(amy, k), tensor_y(apy, k),
                         tensor_x(bmx, k), tensor_x(bpx, k), tensor_y(bmy, k), tensor_y(bpy, k)};
  for (int b = 0; b < 8; ++b) std::copy(blocks[b].begin(), blocks[b].end(), hp.kblocks.begin() + b * ss);

  // cross-section blocks by (K+2)^2 Gauss points
  std::vector<double> gn, gw;
  gauss_legendre(nq, gn, gw);
  std::vector<double> bxv(static_cast<size_t>(n1) * nq), byv(static_cast<size_t>(n1) * nq);
  for (int m = 0; m < n1; ++m)
    for (int g = 0; g < nq; ++g) {
      bxv[m * nq + g] = std::sqrt((2.0 * m + 1.0) / dx) * legendre_value(m, gn[g]);
      byv[m * nq + g] = std::sqrt((2.0 * m + 1.0) / dy) * legendre_value(m, gn[g]);
    }
  hp.sigma_t.assign(ss * hp.ncell, 0.0);
  hp.sigma_s.assign(ss * hp.ncell, 0.0);
  hp.sigma_a.assign(ss * hp.ncell, 0.0);
  std::vector<double> eta(s);
  for (int b = 0; b < hp.ny; ++b)
    for (int a = 0; a < hp.nx; ++a) {
      const int c = b * hp.nx + a;
      double* bs = &hp.sigma_s[ss * c];
      double* ba = &hp.sigma_a[ss * c];
      for (int gy = 0; gy < nq; ++gy) {
        const double y = y_center(b) + 0.5 * dy * gn[gy];
        for (int gx = 0; gx < nq; ++gx) {
          const double x = x_center(a) + 0.5 * dx * gn[gx];
          const double sgs = cfg.sigma_s(x, y), sga = cfg.sigma_a(x, y);
          if (sgs < 0.0 || sga < 0.0) throw std::invalid_argument("assemble_operators: negative cross section");
          const double w = gw[gx] * gw[gy] * 0.25 * dx * dy;
          for (int my = 0; my < n1; ++my)
            for (int mx = 0; mx < n1; ++mx) eta[my * n1 + mx] = bxv[mx * nq + gx] * byv[my * nq + gy];
          // bs += (w ss) (eta eta^T): entry (i, j) += (alpha eta_i) eta_j
          const double ws = w * sgs, wa = w * sga;
          for (int j = 0; j < s; ++j)
            for (int i = 0; i < s; ++i) {
              bs[j * s + i] += (ws * eta[i]) * eta[j];
              ba[j * s + i] += (wa * eta[i]) * eta[j];
            }
        }
      }
      double* bt = &hp.sigma_t[ss * c];
      for (size_t i = 0; i < ss; ++i) bt[i] = bs[i] + ba[i];
    }
  hp.sigma_t_uniform = true;
  for (int c = 1; c < hp.ncell && hp.sigma_t_uniform; ++c)
    if (!std::equal(hp.sigma_t.begin() + ss * c, hp.sigma_t.begin() + ss * (c + 1), hp.sigma_t.begin()))
      hp.sigma_t_uniform = false;

  // source projection
  hp.source.assign(hp.ndof, 0.0);
  for (int b = 0; b < hp.ny; ++b)
    for (int a = 0; a < hp.nx; ++a) {
      const int c = b * hp.nx + a;
      for (int gy = 0; gy < nq; ++gy) {
        const double y = y_center(b) + 0.5 * dy * gn[gy];
        for (int gx = 0; gx < nq; ++gx) {
          const double x = x_center(a) + 0.5 * dx * gn[gx];
          const double w = gw[gx] * gw[gy] * 0.25 * dx * dy * cfg.source(x, y);
          if (w == 0.0) continue;
          for (int my = 0; my < n1; ++my)
            for (int mx = 0; mx < n1; ++mx)
              hp.source[static_cast<size_t>(c) * s + my * n1 + mx] += w * bxv[mx * nq + gx] * byv[my * nq + gy];
        }
      }
    }

  // inflow boundary data (full_rank.cpp:11-39): sampled at the Gauss points first
  hp.bc_any = false;
  hp.bc.clear();
  if (!cfg.boundary_zero && cfg.boundary) {
    double max_abs = 0.0;
    for (int b = 0; b < hp.ny; ++b)
      for (int q = 0; q < nq; ++q) {
        const double y = y_center(b) + 0.5 * dy * gn[q];
        max_abs = std::max(max_abs, std::abs(cfg.boundary(cfg.x_min, y)));
        max_abs = std::max(max_abs, std::abs(cfg.boundary(cfg.x_max, y)));
      }
    for (int a = 0; a < hp.nx; ++a)
      for (int q = 0; q < nq; ++q) {
        const double x = x_center(a) + 0.5 * dx * gn[q];
        max_abs = std::max(max_abs, std::abs(cfg.boundary(x, cfg.y_min)));
        max_abs = std::max(max_abs, std::abs(cfg.boundary(x, cfg.y_max)));
      }
    if (max_abs != 0.0) {
      hp.bc_any = true;
      hp.bc.assign(static_cast<size_t>(hp.n_omega) * hp.ndof, 0.0);
      for (int j = 0; j < hp.n_omega; ++j)
        boundary_vector_general(hp, cfg.boundary, j, &hp.bc[static_cast<size_t>(j) * hp.ndof]);
    }
  }
  hp.sip.clear();  // the DSA is K = 1
  hp.assembly_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace cuda
}  // namespace rtlr
