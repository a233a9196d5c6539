// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp header).
// Restates proj/src/problem.cpp:13-36 (FieldSpec::eval), :111-200 (presets)
// and :461-483 (assemble_problem); adds the BASELINE configs C1-C5 as
// ScalarField callables.
#include <cmath>
#include <cstdio>
#include <memory>

#include "oracle.hpp"

namespace oracle {

namespace {

Field constant(double v) {
  return [v](double, double) { return v; };
}
// proj/src/problem.cpp:18-19
Field gaussian(double amp, double decay, double cx, double cy) {
  return [=](double x, double y) {
    double rx = x - cx, ry = y - cy;
    return amp * std::exp(-decay * (rx * rx + ry * ry));
  };
}
// proj/src/problem.cpp:21-22 (inclusive on both ends)
Field box(double inside, double outside, double x0, double x1, double y0, double y1) {
  return [=](double x, double y) {
    return (x >= x0 && x <= x1 && y >= y0 && y <= y1) ? inside : outside;
  };
}
// proj/src/problem.cpp:23-28
Field radial_transition() {
  return [](double x, double y) {
    double r2 = x * x + y * y;
    if (r2 > 1.0) return 100.0;
    double t = r2 - 2.0;
    return 99.9 * r2 * r2 * t * t + 0.1;
  };
}
// proj/src/problem.cpp:29-33, 85-91
Field lattice_mask(double inside, double outside) {
  static const int cells[8][2] = {{1, 1}, {3, 1}, {1, 3}, {3, 3}, {2, 0}, {0, 2}, {4, 2}, {2, 4}};
  return [=](double x, double y) {
    for (auto& c : cells)
      if (x >= c[0] && x <= c[0] + 1 && y >= c[1] && y <= c[1] + 1) return inside;
    return outside;
  };
}

// 53-bit uniform from mt19937_64 (C4 generator).
double u53(std::mt19937_64& g) { return static_cast<double>(g() >> 11) * 0x1.0p-53; }

struct C4Medium {
  std::vector<double> sig_t, c;  // 64 x 64 patches, patch index py*64+px
  std::vector<int> sq;           // 10 squares: (ax, by) lower-left cell indices
  std::vector<char> src;         // 512 x 512 cell mask
};

std::shared_ptr<C4Medium> make_c4(std::uint64_t seed) {
  auto m = std::make_shared<C4Medium>();
  std::mt19937_64 g(seed);
  m->sig_t.resize(64 * 64);
  m->c.resize(64 * 64);
  for (int p = 0; p < 64 * 64; ++p) {
    const double u1 = u53(g), u2 = u53(g);
    const double z = std::sqrt(-2.0 * std::log(1.0 - u1)) * std::cos(2.0 * M_PI * u2);
    m->sig_t[p] = std::exp(1.5 * z);
    m->c[p] = 0.5 + 0.499 * u53(g);
  }
  m->src.assign(512 * 512, 0);
  for (int k = 0; k < 10; ++k) {
    const int ax = static_cast<int>(u53(g) * 497.0);
    const int by = static_cast<int>(u53(g) * 497.0);
    m->sq.push_back(ax);
    m->sq.push_back(by);
    for (int b = by; b < by + 16; ++b)
      for (int a = ax; a < ax + 16; ++a) m->src[b * 512 + a] = 1;
  }
  return m;
}

int clampi(int v, int hi) { return v < 0 ? 0 : (v > hi ? hi : v); }

}  // namespace

double c5_uniform(std::uint64_t seed, std::uint64_t counter) {
  std::uint64_t z = counter * 0x9E3779B97F4A7C15ull + seed;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return static_cast<double>(z >> 11) * 0x1.0p-53;
}

ProblemSpec make_problem(const std::string& name_in) {
  std::string name = name_in;
  bool full = false;
  if (name.size() > 5 && name.substr(name.size() - 5) == ":full") {
    full = true;
    name = name.substr(0, name.size() - 5);
  }
  ProblemSpec c;
  c.source = constant(0.0);
  c.sigma_a = constant(0.0);
  c.sigma_s = constant(1.0);
  std::string base = name, args;
  auto lp = name.find('(');
  if (lp != std::string::npos) {
    auto rp = name.rfind(')');
    if (rp == std::string::npos || rp < lp)
      throw std::invalid_argument("preset: unbalanced parentheses in '" + name + "'");
    base = name.substr(0, lp);
    args = name.substr(lp + 1, rp - lp - 1);
  }
  if (base == "homogeneous") {  // proj/src/problem.cpp:111-128
    double sigma = 100.0;
    int level = 2;
    if (!args.empty()) {
      char extra = 0;
      if (std::sscanf(args.c_str(), " %lf , %d %c", &sigma, &level, &extra) != 2)
        throw std::invalid_argument("preset: expected homogeneous(sigma_s, L)");
    }
    c.x_min = c.y_min = -1;
    c.x_max = c.y_max = 1;
    c.nx = c.ny = 16 * level;
    c.n_theta = 8 * level;
    c.n_omega_z = 4 * level;
    c.sigma_s = constant(sigma);
    c.source = gaussian(1.0, 100.0, 0.0, 0.0);
    return c;
  }
  if (base == "variable_scattering") {
    c.x_min = c.y_min = -1;
    c.x_max = c.y_max = 1;
    c.nx = c.ny = full ? 80 : 40;
    c.n_theta = full ? 40 : 16;
    c.n_omega_z = full ? 20 : 8;
    c.sigma_s = radial_transition();
    c.source = gaussian(1.0, 100.0, 0.0, 0.0);
    return c;
  }
  if (base == "pin_cell") {
    c.x_min = c.y_min = -1;
    c.x_max = c.y_max = 1;
    c.nx = c.ny = full ? 80 : 40;
    c.n_theta = full ? 32 : 16;
    c.n_omega_z = full ? 16 : 8;
    c.sigma_s = box(0.1, 100.0, -0.5, 0.5, -0.5, 0.5);
    c.source = gaussian(1.0, 100.0, 0.0, 0.0);
    return c;
  }
  if (base == "lattice") {
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
  // ---- BASELINE configs ----
  c.x_min = c.y_min = 0;
  c.x_max = c.y_max = 1;
  if (base == "C1") {
    c.nx = c.ny = 64;
    c.n_theta = 16;
    c.n_omega_z = 8;
    c.sigma_s = constant(0.9);
    c.sigma_a = constant(0.1);
    c.source = box(1.0, 0.0, 0.375, 0.625, 0.375, 0.625);
    c.eps_si_sa = 1e-8;
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
    c.p = 4;
    c.q = 8;
    c.seed = 12345;
    return c;
  }
  if (base == "C3") {
    c.nx = c.ny = 256;
    c.n_theta = 48;
    c.n_omega_z = 24;
    auto absorber = [](double x, double y) {
      int i = clampi(static_cast<int>(x * 7.0), 6), j = clampi(static_cast<int>(y * 7.0), 6);
      return (i + j) % 2 == 1;
    };
    c.sigma_s = [absorber](double x, double y) { return absorber(x, y) ? 0.0 : 1.0; };
    c.sigma_a = [absorber](double x, double y) { return absorber(x, y) ? 10.0 : 0.0; };
    c.source = [](double x, double y) {
      int i = clampi(static_cast<int>(x * 7.0), 6), j = clampi(static_cast<int>(y * 7.0), 6);
      return (i == 3 && j == 3) ? 1.0 : 0.0;
    };
    c.p = 8;
    c.q = 16;
    c.seed = 12345;
    return c;
  }
  if (base == "C4") {
    c.nx = c.ny = 512;
    c.n_theta = 64;
    c.n_omega_z = 32;
    auto med = make_c4(12345);
    c.sigma_s = [med](double x, double y) {
      int p = clampi(static_cast<int>(y * 64.0), 63) * 64 + clampi(static_cast<int>(x * 64.0), 63);
      return med->c[p] * med->sig_t[p];
    };
    c.sigma_a = [med](double x, double y) {
      int p = clampi(static_cast<int>(y * 64.0), 63) * 64 + clampi(static_cast<int>(x * 64.0), 63);
      return (1.0 - med->c[p]) * med->sig_t[p];
    };
    c.source = [med](double x, double y) {
      int a = clampi(static_cast<int>(x * 512.0), 511), b = clampi(static_cast<int>(y * 512.0), 511);
      return med->src[b * 512 + a] ? 1.0 : 0.0;
    };
    c.p = 8;
    c.q = 16;
    c.seed = 12345;
    return c;
  }
  if (base == "C5") {  // isolated sweep medium: sigma_t = 1
    c.nx = c.ny = 256;
    c.n_theta = 32;
    c.n_omega_z = 8;
    c.sigma_s = constant(0.0);
    c.sigma_a = constant(1.0);
    c.source = constant(0.0);
    return c;
  }
  throw std::invalid_argument("unknown preset '" + name_in + "'");
}

// proj/src/problem.cpp:461-483
void assemble_problem(const ProblemSpec& spec, AssembledProblem& out) {
  SpatialMesh mesh = make_mesh(spec.x_min, spec.x_max, spec.y_min, spec.y_max, spec.nx, spec.ny);
  out.space = build_dg_space(mesh, spec.degree);
  out.quad = build_cl_quadrature(spec.n_theta, spec.n_omega_z);
  out.ops = assemble_operators(out.space, spec.sigma_s, spec.sigma_a);
  out.source = project_source(out.space, spec.source);
  if (spec.boundary_zero || !spec.boundary)
    out.bc = BoundaryData{};
  else
    out.bc = build_boundary_data(out.space, out.quad, spec.boundary);
  delete out.dsa;
  out.dsa = nullptr;
  if (spec.use_dsa) out.dsa = new DiffusionSystem(out.space, out.ops, spec.dsa_factor);
}

}  // namespace oracle
