// Host assembly for the B200 compute core (see host.hpp).  Each routine
// cites the reference code it reproduces bit for bit.
#include "host.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>

namespace rtlr {
namespace cuda {

// ------------------------------------------------------------ quadrature
double legendre_value(int n, double x) {  // quadrature.cpp:8-17
  if (n == 0) return 1.0;
  double pm1 = 1.0, p = x;
  for (int k = 2; k <= n; ++k) {
    double pk = ((2.0 * k - 1.0) * x * p - (k - 1.0) * pm1) / k;
    pm1 = p;
    p = pk;
  }
  return p;
}

double legendre_derivative(int n, double x) {  // quadrature.cpp:19-27
  if (n == 0) return 0.0;
  if (std::abs(1.0 - x * x) < 1e-14) {
    double sign = (x > 0.0 || n % 2 == 1) ? 1.0 : -1.0;
    return sign * 0.5 * n * (n + 1.0);
  }
  return n * (legendre_value(n - 1, x) - x * legendre_value(n, x)) / (1.0 - x * x);
}

void gauss_legendre(int n, std::vector<double>& nodes, std::vector<double>& weights) {
  // quadrature.cpp:29-54: Newton on P_n, nodes mirrored exactly.
  if (n < 1) throw std::invalid_argument("gauss_legendre: need at least one node");
  nodes.assign(n, 0.0);
  weights.assign(n, 0.0);
  const int half = (n + 1) / 2;
  for (int i = 0; i < half; ++i) {
    double x = std::cos(M_PI * (i + 0.75) / (n + 0.5));
    for (int it = 0; it < 100; ++it) {
      double p = legendre_value(n, x);
      double dp = legendre_derivative(n, x);
      double d = p / dp;
      x -= d;
      if (std::abs(p) < 1e-15 && std::abs(d) < 1e-15) break;
    }
    double dp = legendre_derivative(n, x);
    double w = 2.0 / ((1.0 - x * x) * dp * dp);
    nodes[n - 1 - i] = x;
    nodes[i] = -x;
    weights[n - 1 - i] = w;
    weights[i] = w;
  }
  if (n % 2 == 1) nodes[half - 1] = 0.0;
}

void build_cl_quadrature(int n_theta, int n_omega_z, std::vector<double>& dirs,
                         std::vector<double>& weights) {
  // quadrature.cpp:56-84: j = j1 * n_omega_z + j2 (azimuth-major).
  if (n_theta < 1 || n_omega_z < 1)
    throw std::invalid_argument("build_cl_quadrature: node counts must be positive");
  std::vector<double> z, wz;
  gauss_legendre(n_omega_z, z, wz);
  const int n = n_theta * n_omega_z;
  dirs.assign(3 * static_cast<size_t>(n), 0.0);
  weights.assign(n, 0.0);
  const double w_theta = 1.0 / n_theta;
  for (int j1 = 0; j1 < n_theta; ++j1) {
    const double theta = (2.0 * j1 + 1.0) * M_PI / n_theta;
    const double c = std::cos(theta), s = std::sin(theta);
    for (int j2 = 0; j2 < n_omega_z; ++j2) {
      const double rho = std::sqrt(1.0 - z[j2] * z[j2]);
      const int j = j1 * n_omega_z + j2;
      dirs[3 * j] = c * rho;
      dirs[3 * j + 1] = s * rho;
      dirs[3 * j + 2] = z[j2];
      weights[j] = w_theta * (0.5 * wz[j2]);
    }
  }
}

// ------------------------------------------------------------ fields / presets
namespace {

Field constant(double v) {
  return [v](double, double) { return v; };
}
Field gaussian(double amp, double decay, double cx, double cy) {  // problem.cpp:18-19
  return [=](double x, double y) {
    double rx = x - cx, ry = y - cy;
    return amp * std::exp(-decay * (rx * rx + ry * ry));
  };
}
Field box(double in, double out, double x0, double x1, double y0, double y1) {  // problem.cpp:21-22
  return [=](double x, double y) { return (x >= x0 && x <= x1 && y >= y0 && y <= y1) ? in : out; };
}
Field radial_transition() {  // problem.cpp:23-28
  return [](double x, double y) {
    double r2 = x * x + y * y;
    if (r2 > 1.0) return 100.0;
    double t = r2 - 2.0;
    return 99.9 * r2 * r2 * t * t + 0.1;
  };
}
Field lattice_mask(double in, double out) {  // problem.cpp:29-33, 85-91
  static const int cells[8][2] = {{1, 1}, {3, 1}, {1, 3}, {3, 3}, {2, 0}, {0, 2}, {4, 2}, {2, 4}};
  return [=](double x, double y) {
    for (auto& c : cells)
      if (x >= c[0] && x <= c[0] + 1 && y >= c[1] && y <= c[1] + 1) return in;
    return out;
  };
}
int clampi(int v, int hi) { return v < 0 ? 0 : (v > hi ? hi : v); }

// C4 heterogeneous medium: mt19937_64(seed), 53-bit uniforms, Box-Muller;
// patches (64 x 64, patch-major) first, then 10 squares (union).
struct C4Medium {
  std::vector<double> sig_t, c;
  std::vector<char> src;
};
std::shared_ptr<C4Medium> make_c4(std::uint64_t seed) {
  auto m = std::make_shared<C4Medium>();
  std::mt19937_64 g(seed);
  auto u53 = [&g] { return static_cast<double>(g() >> 11) * 0x1.0p-53; };
  m->sig_t.resize(4096);
  m->c.resize(4096);
  for (int p = 0; p < 4096; ++p) {
    const double u1 = u53(), u2 = u53();
    const double z = std::sqrt(-2.0 * std::log(1.0 - u1)) * std::cos(2.0 * M_PI * u2);
    m->sig_t[p] = std::exp(1.5 * z);
    m->c[p] = 0.5 + 0.499 * u53();
  }
  m->src.assign(512 * 512, 0);
  for (int k = 0; k < 10; ++k) {
    const int ax = static_cast<int>(u53() * 497.0);
    const int by = static_cast<int>(u53() * 497.0);
    for (int b = by; b < by + 16; ++b)
      for (int a = ax; a < ax + 16; ++a) m->src[b * 512 + a] = 1;
  }
  return m;
}

}  // namespace

ProblemConfig make_config(const std::string& name_in) {
  std::string name = name_in;
  bool full = false;
  if (name.size() > 5 && name.compare(name.size() - 5, 5, ":full") == 0) {
    full = true;
    name.resize(name.size() - 5);
  }
  ProblemConfig c;
  c.preset = name_in;
  c.sigma_s = constant(1.0);
  c.sigma_a = constant(0.0);
  c.source = constant(0.0);
  std::string base = name, args;
  const auto lp = name.find('(');
  if (lp != std::string::npos) {
    const auto rp = name.rfind(')');
    if (rp == std::string::npos || rp < lp)
      throw ConfigError("preset: unbalanced parentheses in '" + name + "'");
    base = name.substr(0, lp);
    args = name.substr(lp + 1, rp - lp - 1);
  }
  if (base == "homogeneous") {  // problem.cpp:111-128, 144-153
    double sigma = 100.0;
    int level = 2;
    if (!args.empty()) {
      char extra = 0;
      if (std::sscanf(args.c_str(), " %lf , %d %c", &sigma, &level, &extra) != 2)
        throw ConfigError("preset: expected homogeneous(sigma_s, L)");
    }
    if (level < 1) throw ConfigError("homogeneous preset: level must be >= 1");
    c.x_min = c.y_min = -1;
    c.x_max = c.y_max = 1;
    c.nx = c.ny = 16 * level;
    c.n_theta = 8 * level;
    c.n_omega_z = 4 * level;
    c.sigma_s = constant(sigma);
    c.source = gaussian(1.0, 100.0, 0.0, 0.0);
    return c;
  }
  if (base == "variable_scattering") {  // problem.cpp:154-167
    c.x_min = c.y_min = -1;
    c.x_max = c.y_max = 1;
    c.nx = c.ny = full ? 80 : 40;
    c.n_theta = full ? 40 : 16;
    c.n_omega_z = full ? 20 : 8;
    c.sigma_s = radial_transition();
    c.source = gaussian(1.0, 100.0, 0.0, 0.0);
    return c;
  }
  if (base == "pin_cell") {  // problem.cpp:168-182
    c.x_min = c.y_min = -1;
    c.x_max = c.y_max = 1;
    c.nx = c.ny = full ? 80 : 40;
    c.n_theta = full ? 32 : 16;
    c.n_omega_z = full ? 16 : 8;
    c.sigma_s = box(0.1, 100.0, -0.5, 0.5, -0.5, 0.5);
    c.source = gaussian(1.0, 100.0, 0.0, 0.0);
    return c;
  }
  if (base == "lattice") {  // problem.cpp:183-197
    c.x_min = c.y_min = 0;
    c.x_max = c.y_max = 5;
    c.nx = c.ny = full ? 80 : 40;
    c.n_theta = full ? 32 : 16;
    c.n_omega_z = full ? 16 : 8;
    c.sigma_a = lattice_mask(100.0, 0.0);
    c.sigma_s = lattice_mask(0.0, 1.0);
    c.source = box(1.0, 0.0, 2.0, 3.0, 2.0, 3.0);
    return c;
  }
  // BASELINE configs; domain [0,1]^2.
  c.x_min = c.y_min = 0;
  c.x_max = c.y_max = 1;
  if (base == "C1") {
    c.nx = c.ny = 64;
    c.n_theta = 16;
    c.n_omega_z = 8;
    c.sigma_s = constant(0.9);
    c.sigma_a = constant(0.1);
    c.source = box(1.0, 0.0, 0.375, 0.625, 0.375, 0.625);
    c.solver.eps_si_sa = 1e-8;
    return c;
  }
  if (base == "C2") {
    c.nx = c.ny = 128;
    c.n_theta = 32;
    c.n_omega_z = 16;
    c.sigma_s = constant(99.9);
    c.sigma_a = constant(0.1);
    c.source = [](double x, double y) {
      return 1.0 + 0.5 * std::sin(2.0 * M_PI * x) * std::sin(2.0 * M_PI * y);
    };
    c.solver.p = 4;
    c.solver.q = 8;
    c.solver.seed = 12345;
    return c;
  }
  if (base == "C3") {
    c.nx = c.ny = 256;
    c.n_theta = 48;
    c.n_omega_z = 24;
    auto absorber = [](double x, double y) {
      const int i = clampi(static_cast<int>(x * 7.0), 6), j = clampi(static_cast<int>(y * 7.0), 6);
      return (i + j) % 2 == 1;
    };
    c.sigma_s = [absorber](double x, double y) { return absorber(x, y) ? 0.0 : 1.0; };
    c.sigma_a = [absorber](double x, double y) { return absorber(x, y) ? 10.0 : 0.0; };
    c.source = [](double x, double y) {
      const int i = clampi(static_cast<int>(x * 7.0), 6), j = clampi(static_cast<int>(y * 7.0), 6);
      return (i == 3 && j == 3) ? 1.0 : 0.0;
    };
    c.solver.p = 8;
    c.solver.q = 16;
    c.solver.seed = 12345;
    return c;
  }
  if (base == "C4") {
    c.nx = c.ny = 512;
    c.n_theta = 64;
    c.n_omega_z = 32;
    auto med = make_c4(12345);
    auto patch = [](double x, double y) {
      return clampi(static_cast<int>(y * 64.0), 63) * 64 + clampi(static_cast<int>(x * 64.0), 63);
    };
    c.sigma_s = [med, patch](double x, double y) {
      const int p = patch(x, y);
      return med->c[p] * med->sig_t[p];
    };
    c.sigma_a = [med, patch](double x, double y) {
      const int p = patch(x, y);
      return (1.0 - med->c[p]) * med->sig_t[p];
    };
    c.source = [med](double x, double y) {
      const int a = clampi(static_cast<int>(x * 512.0), 511), b = clampi(static_cast<int>(y * 512.0), 511);
      return med->src[b * 512 + a] ? 1.0 : 0.0;
    };
    c.solver.p = 8;
    c.solver.q = 16;
    c.solver.seed = 12345;
    return c;
  }
  if (base == "C5") {  // isolated sweep medium, sigma_t = 1
    c.nx = c.ny = 256;
    c.n_theta = 32;
    c.n_omega_z = 8;
    c.sigma_s = constant(0.0);
    c.sigma_a = constant(1.0);
    c.source = constant(0.0);
    return c;
  }
  throw ConfigError("unknown preset '" + name_in + "'");
}

void validate_config(const ProblemConfig& c) {  // problem.cpp:95-107
  if (!(c.x_min < c.x_max) || !(c.y_min < c.y_max)) throw ConfigError("config: empty domain");
  if (c.nx < 1 || c.ny < 1) throw ConfigError("config: cell counts must be positive");
  if (c.n_theta < 1 || c.n_omega_z < 1) throw ConfigError("config: quadrature orders must be positive");
  if (c.degree < 0) throw ConfigError("config: negative polynomial degree");
  const SolverParams& s = c.solver;
  for (double tol : {s.eps_si_sa, s.eps_res, s.eps_diff, s.eps_svd, s.eps_mgs})
    if (!(tol > 0.0)) throw ConfigError("config: tolerances must be positive");
  if (s.p < 1 || s.q < s.p) throw ConfigError("config: need 1 <= p <= q");
  if (s.max_iterations < 1) throw ConfigError("config: max_iterations must be positive");
}

// ------------------------------------------------------------ assembly
namespace {

// operators.cpp:13-57 for K = 1, with the reference's rounding.
void stream_consts(double h, double a_minus[4], double a_plus[4], double b_minus[4],
                   double b_plus[4], double tr[2], double tl[2]) {
  // 2x2 column-major: index (i,j) -> j*2+i
  const double v10 = 2.0 * std::sqrt((2.0 * 1 + 1.0) * (2.0 * 0 + 1.0)) / h;  // d(1,0)
  const double v[4] = {0.0, v10, 0.0, 0.0};
  tr[0] = std::sqrt((2.0 * 0 + 1.0) / h);
  tr[1] = std::sqrt((2.0 * 1 + 1.0) / h);
  tl[0] = tr[0];
  tl[1] = -tr[1];
  for (int j = 0; j < 2; ++j)
    for (int i = 0; i < 2; ++i) {
      a_minus[j * 2 + i] = -v[j * 2 + i] + tr[i] * tr[j];
      a_plus[j * 2 + i] = -v[j * 2 + i] - tl[i] * tl[j];
      b_minus[j * 2 + i] = -tl[i] * tr[j];
      b_plus[j * 2 + i] = tr[i] * tl[j];
    }
}
// tensor_with_identity_x/_y (operators.cpp:61-79) into 4x4 column-major.
void tensor_x4(const double b[4], double out[16]) {
  std::memset(out, 0, 16 * sizeof(double));
  for (int my = 0; my < 2; ++my)
    for (int mx = 0; mx < 2; ++mx)
      for (int lx = 0; lx < 2; ++lx) out[(my * 2 + lx) * 4 + (my * 2 + mx)] = b[lx * 2 + mx];
}
void tensor_y4(const double b[4], double out[16]) {
  std::memset(out, 0, 16 * sizeof(double));
  for (int mx = 0; mx < 2; ++mx)
    for (int my = 0; my < 2; ++my)
      for (int ly = 0; ly < 2; ++ly) out[(ly * 2 + mx) * 4 + (my * 2 + mx)] = b[ly * 2 + my];
}

// diffusion.cpp:15-28 (K = 1, 3-point Gauss)
void stiffness_1d(double h, double st[4]) {
  std::vector<double> nodes, w;
  gauss_legendre(3, nodes, w);
  for (int i = 0; i < 4; ++i) st[i] = 0.0;
  for (int g = 0; g < 3; ++g) {
    double dphi[2];
    for (int m = 0; m < 2; ++m)
      dphi[m] = std::sqrt((2.0 * m + 1.0) / h) * legendre_derivative(m, nodes[g]) * 2.0 / h;
    const double alpha = 0.5 * h * w[g];
    for (int j = 0; j < 2; ++j)
      for (int i = 0; i < 2; ++i) st[j * 2 + i] += (alpha * dphi[i]) * dphi[j];
  }
}
void edge_values(double h, bool right, double v[2]) {  // diffusion.cpp:30-37
  for (int m = 0; m <= 1; ++m) {
    const double p = right ? 1.0 : ((m % 2 == 0) ? 1.0 : -1.0);
    v[m] = std::sqrt((2.0 * m + 1.0) / h) * p;
  }
}
void edge_derivatives(double h, bool right, double v[2]) {  // diffusion.cpp:40-48
  for (int m = 0; m <= 1; ++m) {
    double dp = 0.5 * m * (m + 1.0);
    if (!right && m % 2 == 0) dp = -dp;
    v[m] = std::sqrt((2.0 * m + 1.0) / h) * dp * 2.0 / h;
  }
}
// diffusion.cpp:79-88: e(k,l) = -gu[l] st vt[k] - gt[k] su vu[l] + gamma st su vt[k] vu[l]
void sip_face(const double vt[2], const double gt[2], double st, const double vu[2],
              const double gu[2], double su, double gamma, double e[4]) {
  for (int k = 0; k < 2; ++k)
    for (int l = 0; l < 2; ++l)
      e[l * 2 + k] = -gu[l] * st * vt[k] - gt[k] * su * vu[l] + gamma * st * su * vt[k] * vu[l];
}
void scale2(double a, const double v[2], double o[2]) {
  o[0] = a * v[0];
  o[1] = a * v[1];
}
void add16(double* dst, const double* src) {
  for (int i = 0; i < 16; ++i) dst[i] += src[i];
}

}  // namespace

// SIP-DG diffusion matrix + Sigma_a (diffusion.cpp:90-193) from the
// assembled Sigma_t / Sigma_a blocks and the mesh.
void build_sip(HostProblem& hp) {
  const double dx = hp.dx, dy = hp.dy;
  hp.sip.clear();
  // SIP-DG diffusion matrix + Sigma_a (diffusion.cpp:90-193), in BSR.  The
  // reference sums duplicate triplets in insertion order: volume, x faces
  // (rows b outer, faces af inner), y faces (columns a outer, bf inner),
  // then adds Sigma_a.  For the self block of cell (a,b) that order is
  // volume, left x face, right x face, bottom y face, top y face.
  const double pen = 4.0 * std::max(1 * (1 + 1), 1);
  std::vector<double> d_cell(hp.ncell);
  for (int c = 0; c < hp.ncell; ++c) {
    const double sig = hp.sigma_t[16 * static_cast<size_t>(c)];  // (0,0) entry
    if (!(sig > 0.0)) throw std::runtime_error("build_diffusion: sigma_t must be positive");
    d_cell[c] = 1.0 / (3.0 * sig);
  }
  double stx[4], sty[4], vol[16], voly[16];
  stiffness_1d(dx, stx);
  stiffness_1d(dy, sty);
  tensor_x4(stx, vol);
  tensor_y4(sty, voly);
  for (int i = 0; i < 16; ++i) vol[i] = vol[i] + voly[i];
  double vxl[2], vxr[2], gxl[2], gxr[2], vyl[2], vyr[2], gyl[2], gyr[2];
  edge_values(dx, false, vxl);
  edge_values(dx, true, vxr);
  edge_derivatives(dx, false, gxl);
  edge_derivatives(dx, true, gxr);
  edge_values(dy, false, vyl);
  edge_values(dy, true, vyr);
  edge_derivatives(dy, false, gyl);
  edge_derivatives(dy, true, gyr);
  hp.sip.assign(static_cast<size_t>(hp.ncell) * 80, 0.0);
  auto blk = [&](int c, int slot) { return &hp.sip[(static_cast<size_t>(c) * 5 + slot) * 16]; };
  for (int c = 0; c < hp.ncell; ++c)
    for (int i = 0; i < 16; ++i) blk(c, 0)[i] = d_cell[c] * vol[i];
  // x faces: self-block contributions must be added left face first, then
  // right face; both happen in this (b, af ascending) loop order.
  double e[4], t16[16];
  for (int b = 0; b < hp.ny; ++b)
    for (int af = 0; af <= hp.nx; ++af) {
      const bool has_l = af > 0, has_r = af < hp.nx;
      const int cl = has_l ? b * hp.nx + af - 1 : -1, cr = has_r ? b * hp.nx + af : -1;
      if (has_l && has_r) {
        const double dl = d_cell[cl], dr = d_cell[cr];
        const double wsum = dl + dr, wl = dr / wsum, wr = dl / wsum;
        const double dharm = 2.0 * dl * dr / wsum;
        const double gamma = pen * dharm / dx;
        double fl[2], fr[2];
        scale2(wl * dl, gxr, fl);
        scale2(wr * dr, gxl, fr);
        sip_face(vxr, fl, 1, vxr, fl, 1, gamma, e);
        tensor_x4(e, t16);
        add16(blk(cl, 0), t16);
        sip_face(vxr, fl, 1, vxl, fr, -1, gamma, e);
        tensor_x4(e, t16);
        add16(blk(cl, 2), t16);  // east neighbour of cl
        sip_face(vxl, fr, -1, vxr, fl, 1, gamma, e);
        tensor_x4(e, t16);
        add16(blk(cr, 1), t16);  // west neighbour of cr
        sip_face(vxl, fr, -1, vxl, fr, -1, gamma, e);
        tensor_x4(e, t16);
        add16(blk(cr, 0), t16);
      } else {
        const int c = has_l ? cl : cr;
        const double* v = has_l ? vxr : vxl;
        double g[2];
        if (has_l)
          scale2(d_cell[c], gxr, g);
        else
          scale2(-d_cell[c], gxl, g);
        const double gamma = pen * d_cell[c] / dx;
        sip_face(v, g, 1, v, g, 1, gamma, e);
        tensor_x4(e, t16);
        add16(blk(c, 0), t16);
      }
    }
  for (int a = 0; a < hp.nx; ++a)
    for (int bf = 0; bf <= hp.ny; ++bf) {
      const bool has_b = bf > 0, has_t = bf < hp.ny;
      const int cb = has_b ? (bf - 1) * hp.nx + a : -1, ct = has_t ? bf * hp.nx + a : -1;
      if (has_b && has_t) {
        const double db = d_cell[cb], dt = d_cell[ct];
        const double wsum = db + dt, wb = dt / wsum, wt = db / wsum;
        const double dharm = 2.0 * db * dt / wsum;
        const double gamma = pen * dharm / dy;
        double fb[2], ft[2];
        scale2(wb * db, gyr, fb);
        scale2(wt * dt, gyl, ft);
        sip_face(vyr, fb, 1, vyr, fb, 1, gamma, e);
        tensor_y4(e, t16);
        add16(blk(cb, 0), t16);
        sip_face(vyr, fb, 1, vyl, ft, -1, gamma, e);
        tensor_y4(e, t16);
        add16(blk(cb, 4), t16);  // north neighbour of cb
        sip_face(vyl, ft, -1, vyr, fb, 1, gamma, e);
        tensor_y4(e, t16);
        add16(blk(ct, 3), t16);  // south neighbour of ct
        sip_face(vyl, ft, -1, vyl, ft, -1, gamma, e);
        tensor_y4(e, t16);
        add16(blk(ct, 0), t16);
      } else {
        const int c = has_b ? cb : ct;
        const double* v = has_b ? vyr : vyl;
        double g[2];
        if (has_b)
          scale2(d_cell[c], gyr, g);
        else
          scale2(-d_cell[c], gyl, g);
        const double gamma = pen * d_cell[c] / dy;
        sip_face(v, g, 1, v, g, 1, gamma, e);
        tensor_y4(e, t16);
        add16(blk(c, 0), t16);
      }
    }
  for (int c = 0; c < hp.ncell; ++c) add16(blk(c, 0), &hp.sigma_a[16 * static_cast<size_t>(c)]);
}

void build_stream_consts(HostProblem& hp) {  // operators.cpp:101-112
  double amx[4], apx[4], bmx[4], bpx[4], amy[4], apy[4], bmy[4], bpy[4];
  stream_consts(hp.dx, amx, apx, bmx, bpx, hp.sc.trx_r, hp.sc.trx_l);
  stream_consts(hp.dy, amy, apy, bmy, bpy, hp.sc.try_r, hp.sc.try_l);
  tensor_x4(amx, hp.sc.ax_minus);
  tensor_x4(apx, hp.sc.ax_plus);
  tensor_x4(bmx, hp.sc.bx_minus);
  tensor_x4(bpx, hp.sc.bx_plus);
  tensor_y4(amy, hp.sc.ay_minus);
  tensor_y4(apy, hp.sc.ay_plus);
  tensor_y4(bmy, hp.sc.by_minus);
  tensor_y4(bpy, hp.sc.by_plus);
}

void detect_uniform(HostProblem& hp) {  // every Sigma_t block bitwise identical
  hp.sigma_t_uniform = true;
  for (int c = 1; c < hp.ncell && hp.sigma_t_uniform; ++c)
    if (std::memcmp(&hp.sigma_t[16 * static_cast<size_t>(c)], &hp.sigma_t[0], 16 * sizeof(double)) != 0)
      hp.sigma_t_uniform = false;
}

void assemble(const ProblemConfig& cfg, HostProblem& hp) {
  const auto t0 = std::chrono::steady_clock::now();
  validate_config(cfg);
  if (cfg.degree != 1) {  // sweep / streaming operator only (host_dgk.cpp)
    assemble_general(cfg, hp);
    return;
  }
  hp.cfg = cfg;
  hp.nx = cfg.nx;
  hp.ny = cfg.ny;
  hp.ncell = cfg.nx * cfg.ny;
  hp.ndof = 4 * hp.ncell;
  hp.dx = (cfg.x_max - cfg.x_min) / cfg.nx;  // SpatialMesh::dx (dg_space.hpp:19)
  hp.dy = (cfg.y_max - cfg.y_min) / cfg.ny;
  build_cl_quadrature(cfg.n_theta, cfg.n_omega_z, hp.dirs, hp.weights);
  hp.n_omega = cfg.n_theta * cfg.n_omega_z;
  const double dx = hp.dx, dy = hp.dy;
  auto x_center = [&](int a) { return cfg.x_min + (a + 0.5) * ((cfg.x_max - cfg.x_min) / cfg.nx); };
  auto y_center = [&](int b) { return cfg.y_min + (b + 0.5) * ((cfg.y_max - cfg.y_min) / cfg.ny); };

  build_stream_consts(hp);

  // Cross-section blocks by 3x3 Gauss points (operators.cpp:137-181).
  std::vector<double> gn, gw;
  gauss_legendre(3, gn, gw);
  double bxv[2][3], byv[2][3];
  for (int m = 0; m < 2; ++m)
    for (int g = 0; g < 3; ++g) {
      bxv[m][g] = std::sqrt((2.0 * m + 1.0) / dx) * legendre_value(m, gn[g]);
      byv[m][g] = std::sqrt((2.0 * m + 1.0) / dy) * legendre_value(m, gn[g]);
    }
  hp.sigma_t.assign(16 * static_cast<size_t>(hp.ncell), 0.0);
  hp.sigma_s.assign(16 * static_cast<size_t>(hp.ncell), 0.0);
  hp.sigma_a.assign(16 * static_cast<size_t>(hp.ncell), 0.0);
  for (int b = 0; b < hp.ny; ++b)
    for (int a = 0; a < hp.nx; ++a) {
      const int c = b * hp.nx + a;
      double* bs = &hp.sigma_s[16 * static_cast<size_t>(c)];
      double* ba = &hp.sigma_a[16 * static_cast<size_t>(c)];
      for (int gy = 0; gy < 3; ++gy) {
        const double y = y_center(b) + 0.5 * dy * gn[gy];
        for (int gx = 0; gx < 3; ++gx) {
          const double x = x_center(a) + 0.5 * dx * gn[gx];
          const double ss = cfg.sigma_s(x, y), sa = cfg.sigma_a(x, y);
          if (ss < 0.0 || sa < 0.0) throw std::invalid_argument("assemble_operators: negative cross section");
          const double w = gw[gx] * gw[gy] * 0.25 * dx * dy;
          double eta[4];
          for (int my = 0; my < 2; ++my)
            for (int mx = 0; mx < 2; ++mx) eta[my * 2 + mx] = bxv[mx][gx] * byv[my][gy];
          const double ws = w * ss, wa = w * sa;
          for (int j = 0; j < 4; ++j)
            for (int i = 0; i < 4; ++i) {
              bs[j * 4 + i] += (ws * eta[i]) * eta[j];
              ba[j * 4 + i] += (wa * eta[i]) * eta[j];
            }
        }
      }
      double* bt = &hp.sigma_t[16 * static_cast<size_t>(c)];
      for (int i = 0; i < 16; ++i) bt[i] = bs[i] + ba[i];
    }
  detect_uniform(hp);

  // Source projection (operators.cpp:191-225).
  hp.source.assign(hp.ndof, 0.0);
  for (int b = 0; b < hp.ny; ++b)
    for (int a = 0; a < hp.nx; ++a) {
      const int c = b * hp.nx + a;
      for (int gy = 0; gy < 3; ++gy) {
        const double y = y_center(b) + 0.5 * dy * gn[gy];
        for (int gx = 0; gx < 3; ++gx) {
          const double x = x_center(a) + 0.5 * dx * gn[gx];
          const double w = gw[gx] * gw[gy] * 0.25 * dx * dy * cfg.source(x, y);
          if (w == 0.0) continue;
          for (int my = 0; my < 2; ++my)
            for (int mx = 0; mx < 2; ++mx) hp.source[c * 4 + my * 2 + mx] += w * bxv[mx][gx] * byv[my][gy];
        }
      }
    }

  // Inflow boundary data (full_rank.cpp:11-39).
  hp.bc_any = false;
  hp.bc.clear();
  if (!cfg.boundary_zero && cfg.boundary) {
    double max_abs = 0.0;
    for (int b = 0; b < hp.ny; ++b)
      for (int q = 0; q < 3; ++q) {
        const double y = y_center(b) + 0.5 * dy * gn[q];
        max_abs = std::max(max_abs, std::abs(cfg.boundary(cfg.x_min, y)));
        max_abs = std::max(max_abs, std::abs(cfg.boundary(cfg.x_max, y)));
      }
    for (int a = 0; a < hp.nx; ++a)
      for (int q = 0; q < 3; ++q) {
        const double x = x_center(a) + 0.5 * dx * gn[q];
        max_abs = std::max(max_abs, std::abs(cfg.boundary(x, cfg.y_min)));
        max_abs = std::max(max_abs, std::abs(cfg.boundary(x, cfg.y_max)));
      }
    if (max_abs != 0.0) {
      hp.bc_any = true;
      hp.bc.assign(static_cast<size_t>(hp.n_omega) * hp.ndof, 0.0);
      for (int j = 0; j < hp.n_omega; ++j)
        boundary_vector(hp, cfg.boundary, j, &hp.bc[static_cast<size_t>(j) * hp.ndof]);
    }
  }

  hp.sip.clear();
  if (cfg.solver.use_dsa) build_sip(hp);
  hp.assembly_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

void assemble_arrays(const ProblemArrays& in, HostProblem& hp) {
  const auto t0 = std::chrono::steady_clock::now();
  if (in.nx < 1 || in.ny < 1) throw std::invalid_argument("problem_upload: mesh must have at least one cell");
  if (!(in.x_max > in.x_min) || !(in.y_max > in.y_min)) throw std::invalid_argument("problem_upload: empty domain");
  if (in.n_omega < 1) throw std::invalid_argument("problem_upload: need at least one direction");
  if (in.n_theta < 0 || in.n_omega_z < 0 ||
      ((in.n_theta > 0 || in.n_omega_z > 0) && in.n_theta * in.n_omega_z != in.n_omega))
    throw std::invalid_argument("problem_upload: n_theta * n_omega_z must equal n_omega");
  if (!in.dirs || !in.weights || !in.sigma_t || !in.sigma_s || !in.source)
    throw std::invalid_argument("problem_upload: dirs, weights, sigma_t, sigma_s and source are required");
  ProblemConfig& c = hp.cfg;
  c = ProblemConfig{};
  c.preset = "uploaded";
  c.x_min = in.x_min;
  c.x_max = in.x_max;
  c.y_min = in.y_min;
  c.y_max = in.y_max;
  c.nx = in.nx;
  c.ny = in.ny;
  // an unstructured direction set is one azimuthal line (partition_angles
  // then deals single directions)
  c.n_theta = in.n_theta > 0 ? in.n_theta : in.n_omega;
  c.n_omega_z = in.n_omega_z > 0 ? in.n_omega_z : 1;
  c.solver = in.solver;
  c.solver.use_dsa = in.use_dsa;
  c.boundary_zero = in.boundary == nullptr;
  hp.nx = in.nx;
  hp.ny = in.ny;
  hp.ncell = in.nx * in.ny;
  hp.ndof = 4 * hp.ncell;
  hp.dx = (in.x_max - in.x_min) / in.nx;
  hp.dy = (in.y_max - in.y_min) / in.ny;
  hp.n_omega = in.n_omega;
  const size_t nb = 16 * static_cast<size_t>(hp.ncell);
  hp.dirs.assign(in.dirs, in.dirs + 3 * static_cast<size_t>(in.n_omega));
  hp.weights.assign(in.weights, in.weights + in.n_omega);
  for (double v : hp.dirs)
    if (!std::isfinite(v)) throw std::invalid_argument("problem_upload: non-finite direction");
  build_stream_consts(hp);
  hp.sigma_t.assign(in.sigma_t, in.sigma_t + nb);
  hp.sigma_s.assign(in.sigma_s, in.sigma_s + nb);
  if (in.sigma_a) {
    hp.sigma_a.assign(in.sigma_a, in.sigma_a + nb);
  } else {
    hp.sigma_a.resize(nb);
    for (size_t i = 0; i < nb; ++i) hp.sigma_a[i] = hp.sigma_t[i] - hp.sigma_s[i];
  }
  detect_uniform(hp);
  hp.source.assign(in.source, in.source + hp.ndof);
  hp.bc_any = false;
  hp.bc.clear();
  if (in.boundary) {
    const size_t nbc = static_cast<size_t>(hp.n_omega) * hp.ndof;
    double max_abs = 0.0;
    for (size_t i = 0; i < nbc; ++i) max_abs = std::max(max_abs, std::abs(in.boundary[i]));
    if (max_abs != 0.0) {  // BoundaryData stays empty for a zero datum (full_rank.cpp:32)
      hp.bc_any = true;
      hp.bc.assign(in.boundary, in.boundary + nbc);
    }
  }
  hp.sip.clear();
  if (in.sip)
    hp.sip.assign(in.sip, in.sip + 80 * static_cast<size_t>(hp.ncell));
  else if (in.use_dsa)
    build_sip(hp);
  hp.assembly_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

void boundary_vector(const HostProblem& hp, const Field& g, int angle, double* out) {
  // operators.cpp:227-281
  if (angle < 0 || angle >= hp.n_omega) throw std::invalid_argument("boundary_vector: angle index out of range");
  const ProblemConfig& cfg = hp.cfg;
  const double dx = hp.dx, dy = hp.dy;
  const double omx = hp.dirs[3 * angle], omy = hp.dirs[3 * angle + 1];
  std::vector<double> gn, gw;
  gauss_legendre(3, gn, gw);
  const double trx_l[2] = {hp.sc.trx_l[0], hp.sc.trx_l[1]}, trx_r[2] = {hp.sc.trx_r[0], hp.sc.trx_r[1]};
  const double try_l[2] = {hp.sc.try_l[0], hp.sc.try_l[1]}, try_r[2] = {hp.sc.try_r[0], hp.sc.try_r[1]};
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
  auto add_x_edge = [&](int a, double x_edge, const double* trx, double coeff) {
    for (int b = 0; b < hp.ny; ++b) {
      const int c = b * hp.nx + a;
      for (int q = 0; q < 3; ++q) {
        const double y = y_center(b) + 0.5 * dy * gn[q];
        const double w = coeff * gw[q] * 0.5 * dy * g(x_edge, y);
        if (w == 0.0) continue;
        for (int my = 0; my < 2; ++my) {
          const double by = basis_y(my, b, y);
          for (int mx = 0; mx < 2; ++mx) out[c * 4 + my * 2 + mx] += w * trx[mx] * by;
        }
      }
    }
  };
  auto add_y_edge = [&](int b, double y_edge, const double* tryv, double coeff) {
    for (int a = 0; a < hp.nx; ++a) {
      const int c = b * hp.nx + a;
      for (int q = 0; q < 3; ++q) {
        const double x = x_center(a) + 0.5 * dx * gn[q];
        const double w = coeff * gw[q] * 0.5 * dx * g(x, y_edge);
        if (w == 0.0) continue;
        for (int mx = 0; mx < 2; ++mx) {
          const double bx = basis_x(mx, a, x);
          for (int my = 0; my < 2; ++my) out[c * 4 + my * 2 + mx] += w * tryv[my] * bx;
        }
      }
    }
  };
  if (omx > 0.0) add_x_edge(0, cfg.x_min, trx_l, omx);
  if (omx < 0.0) add_x_edge(hp.nx - 1, cfg.x_max, trx_r, -omx);
  if (omy > 0.0) add_y_edge(0, cfg.y_min, try_l, omy);
  if (omy < 0.0) add_y_edge(hp.ny - 1, cfg.y_max, try_r, -omy);
}

// ------------------------------------------------------------ rng
std::uint64_t SubsampleRng::draw_below(std::uint64_t n) {  // low_rank.cpp:15-26
  if (n == 0) throw std::invalid_argument("draw_below: empty range");
  std::uint64_t mask = ~std::uint64_t{0};
  const std::uint64_t limit = n - 1;
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
  count = std::min<int>(count, static_cast<int>(pool.size()));  // low_rank.cpp:28-37
  for (int i = 0; i < count; ++i) {
    const int j = i + static_cast<int>(draw_below(pool.size() - i));
    std::swap(pool[i], pool[j]);
  }
  pool.resize(count);
  return pool;
}

std::vector<int> partition_angles(int n_theta, int n_omega_z, int nranks, int rank) {
  if (n_theta < 1 || n_omega_z < 1 || nranks < 1 || rank < 0 || rank >= nranks)
    throw std::invalid_argument("partition_angles: bad argument");
  std::vector<int> out;
  const int half = (n_omega_z + 1) / 2;
  int u = 0;
  for (int j2 = 0; j2 < half; ++j2)
    for (int j1 = 0; j1 < n_theta; ++j1, ++u) {
      if (u % nranks != rank) continue;
      const int a = j1 * n_omega_z + j2, b = j1 * n_omega_z + (n_omega_z - 1 - j2);
      out.push_back(a);
      if (b != a) out.push_back(b);
    }
  return out;
}

ShardBlock shard_block(int m, int nranks, int rank) {
  if (m < 0 || nranks < 1 || rank < 0 || rank >= nranks) throw std::invalid_argument("shard_block: bad argument");
  ShardBlock b;
  b.bsz = (m + nranks - 1) / nranks;
  b.begin = std::min(m, rank * b.bsz);
  b.end = std::min(m, b.begin + b.bsz);
  return b;
}

int truncation_rank(const std::vector<double>& s, double eps_svd) {  // low_rank.cpp:254-266
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

}  // namespace cuda
}  // namespace rtlr
