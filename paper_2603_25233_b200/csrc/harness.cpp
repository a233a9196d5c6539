// Run harness (see harness.hpp): config text format, run driver with the
// FR-vs-LR comparison, metrics / history / flux writers.
#include "harness.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <sstream>
#include <stdexcept>

namespace rtlr {
namespace cuda {

namespace {

std::string fmt(double v) {  // report.cpp:15-19, problem.cpp:236-240
  char buf[40];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}

// FieldSpec (problem.hpp:22-47) and its eval (problem.cpp:13-36).
struct Spec {
  enum Kind { Constant, Gaussian, Box, RadialTransition, LatticeMask };
  Kind kind = Constant;
  double value = 0.0, outside = 0.0, x0 = 0.0, x1 = 0.0, y0 = 0.0, y1 = 0.0, decay = 0.0, cx = 0.0, cy = 0.0;
};
Spec constant_spec(double v) {
  Spec s;
  s.value = v;
  return s;
}
Spec gaussian_spec(double amp, double decay, double cx, double cy) {
  Spec s;
  s.kind = Spec::Gaussian;
  s.value = amp;
  s.decay = decay;
  s.cx = cx;
  s.cy = cy;
  return s;
}
Spec box_spec(double in, double out, double x0, double x1, double y0, double y1) {
  Spec s;
  s.kind = Spec::Box;
  s.value = in;
  s.outside = out;
  s.x0 = x0;
  s.x1 = x1;
  s.y0 = y0;
  s.y1 = y1;
  return s;
}
Spec lattice_spec(double in, double out) {
  Spec s;
  s.kind = Spec::LatticeMask;
  s.value = in;
  s.outside = out;
  return s;
}

Field field_of(const Spec& s) {
  switch (s.kind) {
    case Spec::Constant: {
      const double v = s.value;
      return [v](double, double) { return v; };
    }
    case Spec::Gaussian:
      return [s](double x, double y) {
        const double rx = x - s.cx, ry = y - s.cy;
        return s.value * std::exp(-s.decay * (rx * rx + ry * ry));
      };
    case Spec::Box:  // inclusive on both ends (problem.cpp:21-22)
      return [s](double x, double y) {
        return (x >= s.x0 && x <= s.x1 && y >= s.y0 && y <= s.y1) ? s.value : s.outside;
      };
    case Spec::RadialTransition:
      return [](double x, double y) {
        const double r2 = x * x + y * y;
        if (r2 > 1.0) return 100.0;
        const double t = r2 - 2.0;
        return 99.9 * r2 * r2 * t * t + 0.1;
      };
    case Spec::LatticeMask:
      return [s](double x, double y) {  // lattice_absorber_cells (problem.cpp:87-93)
        static const int cells[8][2] = {{1, 1}, {3, 1}, {1, 3}, {3, 3}, {2, 0}, {0, 2}, {4, 2}, {2, 4}};
        for (const auto& c : cells)
          if (x >= c[0] && x <= c[0] + 1 && y >= c[1] && y <= c[1] + 1) return s.value;
        return s.outside;
      };
  }
  return [](double, double) { return 0.0; };
}

Spec::Kind kind_from_name(const std::string& s) {  // problem.cpp:258-265
  if (s == "constant") return Spec::Constant;
  if (s == "gaussian") return Spec::Gaussian;
  if (s == "box") return Spec::Box;
  if (s == "radial_transition") return Spec::RadialTransition;
  if (s == "lattice_mask") return Spec::LatticeMask;
  throw ConfigError("unknown field kind '" + s + "'");
}

// The reference presets' fields as FieldSpecs (make_preset,
// problem.cpp:109-199), so field keys after a preset line modify them as in
// the reference.  Fields are ordered sigma_s, sigma_a, source, boundary.
bool preset_specs(const std::string& name_in, Spec out[4]) {
  std::string name = name_in;
  if (name.size() > 5 && name.compare(name.size() - 5, 5, ":full") == 0) name.resize(name.size() - 5);
  const std::string base = name.substr(0, name.find('('));
  out[3] = constant_spec(0.0);
  if (base == "homogeneous") {
    double sigma = 100.0;
    int level = 2;
    const auto lp = name.find('(');
    if (lp != std::string::npos) std::sscanf(name.c_str() + lp + 1, " %lf , %d", &sigma, &level);
    out[0] = constant_spec(sigma);
    out[1] = constant_spec(0.0);
    out[2] = gaussian_spec(1.0, 100.0, 0.0, 0.0);
    return true;
  }
  if (base == "variable_scattering") {
    out[0] = Spec();
    out[0].kind = Spec::RadialTransition;
    out[1] = constant_spec(0.0);
    out[2] = gaussian_spec(1.0, 100.0, 0.0, 0.0);
    return true;
  }
  if (base == "pin_cell") {
    out[0] = box_spec(0.1, 100.0, -0.5, 0.5, -0.5, 0.5);
    out[1] = constant_spec(0.0);
    out[2] = gaussian_spec(1.0, 100.0, 0.0, 0.0);
    return true;
  }
  if (base == "lattice") {
    out[0] = lattice_spec(0.0, 1.0);
    out[1] = lattice_spec(100.0, 0.0);
    out[2] = box_spec(1.0, 0.0, 2.0, 3.0, 2.0, 3.0);
    return true;
  }
  return false;  // the BASELINE configs C1-C5 build their fields programmatically
}

std::string trim(const std::string& s) {
  const auto b = s.find_first_not_of(" \t\r\n");
  if (b == std::string::npos) return "";
  const auto e = s.find_last_not_of(" \t\r\n");
  return s.substr(b, e - b + 1);
}

double parse_double(const std::string& v, const std::string& key) {  // problem.cpp:342-352
  try {
    std::size_t pos = 0;
    const double d = std::stod(v, &pos);
    if (pos != v.size()) throw std::invalid_argument(v);
    return d;
  } catch (const std::exception&) {
    throw ConfigError("config: bad number '" + v + "' for " + key);
  }
}

long long parse_int(const std::string& v, const std::string& key) {  // problem.cpp:354-364
  try {
    std::size_t pos = 0;
    const long long i = std::stoll(v, &pos);
    if (pos != v.size()) throw std::invalid_argument(v);
    return i;
  } catch (const std::exception&) {
    throw ConfigError("config: bad integer '" + v + "' for " + key);
  }
}

bool apply_field_key(Spec& f, const std::string& fk, const std::string& value, const std::string& key) {
  if (fk == "kind") f.kind = kind_from_name(value);
  else if (fk == "value") f.value = parse_double(value, key);
  else if (fk == "outside") f.outside = parse_double(value, key);
  else if (fk == "x0") f.x0 = parse_double(value, key);
  else if (fk == "x1") f.x1 = parse_double(value, key);
  else if (fk == "y0") f.y0 = parse_double(value, key);
  else if (fk == "y1") f.y1 = parse_double(value, key);
  else if (fk == "decay") f.decay = parse_double(value, key);
  else if (fk == "center_x") f.cx = parse_double(value, key);
  else if (fk == "center_y") f.cy = parse_double(value, key);
  else return false;
  return true;
}

// The preset name as the reference records it (homogeneous_preset formats
// its arguments with %g, problem.cpp:113-114).
std::string canonical_preset(const std::string& name) {
  if (name.rfind("homogeneous", 0) == 0 && name.find(':') == std::string::npos) {
    double sigma = 100.0;
    int level = 2;
    const auto lp = name.find('(');
    if (lp != std::string::npos) std::sscanf(name.c_str() + lp + 1, " %lf , %d", &sigma, &level);
    char buf[64];
    std::snprintf(buf, sizeof buf, "homogeneous(%g,%d)", sigma, level);
    return buf;
  }
  return name;
}

}  // namespace

RunMode run_mode_from_name(const std::string& s) {
  if (s == "full") return RunMode::Full;
  if (s == "lowrank") return RunMode::LowRank;
  if (s == "both") return RunMode::Both;
  throw ConfigError("unknown run mode '" + s + "'");
}

const char* run_mode_name(RunMode m) {
  switch (m) {
    case RunMode::Full: return "full";
    case RunMode::LowRank: return "lowrank";
    case RunMode::Both: return "both";
  }
  return "both";
}

RunConfig parse_config_text(const std::string& text) {
  RunConfig rc;
  // no preset: the ProblemConfig defaults (problem.hpp:69-81)
  Spec cur[4] = {constant_spec(1.0), constant_spec(0.0), constant_spec(0.0), constant_spec(0.0)};
  bool specs_known = true, touched[4] = {false, false, false, false};
  std::string preset;
  std::istringstream is(text);
  std::string line;
  int lineno = 0;
  while (std::getline(is, line)) {
    ++lineno;
    const auto hash = line.find('#');
    if (hash != std::string::npos) line = line.substr(0, hash);
    line = trim(line);
    if (line.empty()) continue;
    const auto eq = line.find('=');
    if (eq == std::string::npos) throw ConfigError("config line " + std::to_string(lineno) + ": expected key = value");
    const std::string key = trim(line.substr(0, eq)), value = trim(line.substr(eq + 1));
    if (key == "preset") {  // resets every field it covers; solver and mode kept
      const SolverParams keep = rc.cfg.solver;
      rc.cfg = make_config(value);
      rc.cfg.solver = keep;
      rc.cfg.preset = canonical_preset(value);
      preset = value;
      specs_known = preset_specs(value, cur);
      for (bool& t : touched) t = false;
      continue;
    }
    const auto dot = key.find('.');
    const std::string section = dot == std::string::npos ? key : key.substr(0, dot);
    const std::string rest = dot == std::string::npos ? "" : key.substr(dot + 1);
    ProblemConfig& c = rc.cfg;
    auto unknown = [&]() { return ConfigError("config: unknown key '" + key + "'"); };
    if (section == "domain") {
      if (rest == "x_min") c.x_min = parse_double(value, key);
      else if (rest == "x_max") c.x_max = parse_double(value, key);
      else if (rest == "y_min") c.y_min = parse_double(value, key);
      else if (rest == "y_max") c.y_max = parse_double(value, key);
      else throw unknown();
    } else if (section == "mesh") {
      if (rest == "nx") c.nx = static_cast<int>(parse_int(value, key));
      else if (rest == "ny") c.ny = static_cast<int>(parse_int(value, key));
      else throw unknown();
    } else if (section == "quadrature") {
      if (rest == "n_theta") c.n_theta = static_cast<int>(parse_int(value, key));
      else if (rest == "n_omega_z") c.n_omega_z = static_cast<int>(parse_int(value, key));
      else throw unknown();
    } else if (section == "space") {
      if (rest == "degree") c.degree = static_cast<int>(parse_int(value, key));
      else throw unknown();
    } else if (section == "sigma_s" || section == "sigma_a" || section == "source" || section == "boundary") {
      const int f = section == "sigma_s" ? 0 : section == "sigma_a" ? 1 : section == "source" ? 2 : 3;
      if (!specs_known)
        throw ConfigError("config: '" + key + "': the fields of preset '" + preset +
                          "' are built programmatically and take no field keys");
      if (!apply_field_key(cur[f], rest, value, key)) throw unknown();
      touched[f] = true;
    } else if (section == "solver") {
      SolverParams& s = c.solver;
      if (rest == "eps_si_sa") s.eps_si_sa = parse_double(value, key);
      else if (rest == "eps_res") s.eps_res = parse_double(value, key);
      else if (rest == "eps_diff") s.eps_diff = parse_double(value, key);
      else if (rest == "eps_svd") s.eps_svd = parse_double(value, key);
      else if (rest == "eps_mgs") s.eps_mgs = parse_double(value, key);
      else if (rest == "p") s.p = static_cast<int>(parse_int(value, key));
      else if (rest == "q") s.q = static_cast<int>(parse_int(value, key));
      else if (rest == "seed") s.seed = static_cast<std::uint64_t>(parse_int(value, key));
      else if (rest == "max_iterations") s.max_iterations = static_cast<int>(parse_int(value, key));
      else if (rest == "use_dsa") s.use_dsa = parse_int(value, key) != 0;
      else if (rest == "store_psi") s.store_psi = parse_int(value, key) != 0;
      else if (rest == "build_factors") s.build_factors = parse_int(value, key) != 0;
      else throw unknown();
    } else if (section == "run") {
      if (rest == "mode") rc.mode = run_mode_from_name(value);
      else throw unknown();
    } else {
      throw unknown();
    }
  }
  // Fields: a preset's own callables unless a field key modified the
  // field; without a preset line every field comes from its FieldSpec.
  ProblemConfig& c = rc.cfg;
  Field* dst[4] = {&c.sigma_s, &c.sigma_a, &c.source, &c.boundary};
  for (int f = 0; f < 4; ++f)
    if (touched[f] || preset.empty()) *dst[f] = field_of(cur[f]);
  if (touched[3] || preset.empty()) c.boundary_zero = cur[3].kind == Spec::Constant && cur[3].value == 0.0;
  validate_config(c);
  return rc;
}

RunConfig load_config_file(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw ConfigError("cannot open config file '" + path + "'");
  std::ostringstream ss;
  ss << in.rdbuf();
  return parse_config_text(ss.str());
}

RunResult run_config(const RunConfig& rc, int device) {
  Problem P(rc.cfg, device);
  return run_assembled(rc, P);
}

bool all_converged(const RunResult& r) {
  return (!r.has_full || r.full.converged) && (!r.has_low || r.low.converged);
}

namespace {
int lr_rank(const SolveReport& low) {
  return low.has_factors ? low.factors.rank : (low.history.empty() ? 0 : low.history.back().rank);
}
}  // namespace

std::string run_summary(const RunResult& r) {
  char buf[512];
  std::string out = "run " + r.run_id + "\n";
  if (r.has_full) {
    std::snprintf(buf, sizeof buf, "  full-rank : iterations %d%s, solve %.3fs, psi DOFs %lld\n", r.full.iterations,
                  r.full.converged ? "" : " (not converged)", r.full.solve_seconds, r.full.psi_dofs);
    out += buf;
  }
  if (r.has_low) {
    const double os_ratio = r.low.history.empty() ? 0.0 : r.low.history.back().oversampling;
    std::snprintf(buf, sizeof buf,
                  "  low-rank  : iterations %d%s, rank %d, oversampling %.4f, solve %.3fs, psi DOFs %lld\n",
                  r.low.iterations, r.low.converged ? "" : " (not converged)", lr_rank(r.low), os_ratio,
                  r.low.solve_seconds, r.low.psi_dofs);
    out += buf;
  }
  if (r.has_comparison) {
    std::snprintf(buf, sizeof buf, "  compare   : speedup %.3fx, compression %.2f%%, |phi_LR-phi_FR|_2 %.3e",
                  r.comparison.speedup, 100.0 * r.comparison.compression_ratio, r.comparison.phi_diff_two_norm);
    out += buf;
    if (r.comparison.has_psi_diff) {
      std::snprintf(buf, sizeof buf, ", |psi_LR-psi_FR|_2 %.3e", r.comparison.psi_diff_two_norm);
      out += buf;
    }
    out += "\n";
  }
  return out;
}

std::string batch_summary(const std::vector<RunResult>& results) {
  int n_lr = 0;
  double rank_mean = 0, rank_sq = 0, speed_mean = 0, phi_mean = 0;
  for (const RunResult& r : results) {
    if (!r.has_low) continue;
    ++n_lr;
    const double rank = lr_rank(r.low);
    rank_mean += rank;
    rank_sq += rank * rank;
    if (r.has_comparison) {
      speed_mean += r.comparison.speedup;
      phi_mean += r.comparison.phi_diff_two_norm;
    }
  }
  if (n_lr <= 1) return "";
  rank_mean /= n_lr;
  const double sd = std::sqrt(std::max(0.0, rank_sq / n_lr - rank_mean * rank_mean));
  char buf[256];
  std::snprintf(buf, sizeof buf, "batch: %d low-rank runs, rank %.2f (+-%.2f)", n_lr, rank_mean, sd);
  std::string out = buf;
  if (speed_mean > 0) {
    std::snprintf(buf, sizeof buf, ", mean speedup %.3fx", speed_mean / n_lr);
    out += buf;
  }
  if (phi_mean > 0) {
    std::snprintf(buf, sizeof buf, ", mean |phi_LR-phi_FR|_2 %.3e", phi_mean / n_lr);
    out += buf;
  }
  return out + "\n";
}

RunResult run_assembled(const RunConfig& rc, Problem& P) {
  RunResult r;
  r.config = rc;
  const std::string preset = rc.cfg.preset.empty() ? "custom" : rc.cfg.preset;
  r.run_id = preset + "-seed" + std::to_string(rc.cfg.solver.seed);
  r.assembly_seconds = P.host().assembly_seconds;
  const SolverParams& s = rc.cfg.solver;
  if (rc.mode == RunMode::Full || rc.mode == RunMode::Both) {  // full_options (report.cpp:21-28)
    FullRankOptions o;
    o.eps_si_sa = s.eps_si_sa;
    o.max_iterations = s.max_iterations;
    o.use_dsa = s.use_dsa;
    o.store_psi = s.store_psi;
    r.full = P.solve_full_rank(o);
    r.has_full = true;
  }
  if (rc.mode == RunMode::LowRank || rc.mode == RunMode::Both) {  // low_options (report.cpp:30-44)
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
    r.low = P.solve_low_rank(o);
    r.has_low = true;
  }
  if (r.has_full && r.has_low) {  // compare_runs (report.cpp:60-74)
    const long long nx = P.host().ndof, nom = P.host().n_omega;
    RunComparison& c = r.comparison;
    c.speedup = r.low.solve_seconds > 0.0 ? r.full.solve_seconds / r.low.solve_seconds : 0.0;
    c.compression_ratio = static_cast<double>(r.low.psi_dofs) / (static_cast<double>(nx) * nom);
    double acc = 0.0;
    for (long long i = 0; i < nx; ++i) {
      const double d = r.low.phi[i] - r.full.phi[i];
      acc += d * d;
    }
    c.phi_diff_two_norm = std::sqrt(acc);
    if (r.full.has_psi && r.low.has_factors) {
      const int rank = r.low.factors.rank;
      DBuf<double> ps, x, sv, v;
      ps.upload(r.full.psi.data(), r.full.psi.size(), P.stream());
      x.upload(r.low.factors.X.data(), r.low.factors.X.size(), P.stream());
      sv.upload(r.low.factors.S.data(), r.low.factors.S.size(), P.stream());
      v.upload(r.low.factors.V.data(), r.low.factors.V.size(), P.stream());
      c.psi_diff_two_norm = P.psi_difference(ps.get(), x.get(), sv.get(), v.get(), rank);
      c.has_psi_diff = true;
    }
    r.has_comparison = true;
  }
  return r;
}

namespace {

// write_flux_file (report.cpp:101-113): cell means phi_c0 / sqrt(dx dy) at
// the cell centres, row by row.
void write_flux_file(const std::string& path, const ProblemConfig& cfg, const std::vector<double>& phi, bool clamp) {
  std::ofstream os(path);
  if (!os) throw std::runtime_error("cannot write '" + path + "'");
  const double dx = (cfg.x_max - cfg.x_min) / cfg.nx, dy = (cfg.y_max - cfg.y_min) / cfg.ny;
  const int per = (cfg.degree + 1) * (cfg.degree + 1);
  for (int b = 0; b < cfg.ny; ++b)
    for (int a = 0; a < cfg.nx; ++a) {
      double v = phi[static_cast<size_t>(b * cfg.nx + a) * per] / std::sqrt(dx * dy);
      if (clamp) v = std::max(v, 1e-16);
      os << fmt(cfg.x_min + (a + 0.5) * dx) << " " << fmt(cfg.y_min + (b + 0.5) * dy) << " " << fmt(v) << "\n";
    }
}

}  // namespace

void write_outputs(const std::vector<RunResult>& results, const std::string& out_dir, bool log_export) {
  namespace fs = std::filesystem;
  fs::create_directories(out_dir);
  {
    std::ofstream os(out_dir + "/metrics.csv");
    if (!os) throw std::runtime_error("cannot write metrics.csv in '" + out_dir + "'");
    os << "run_id,preset,mode,seed,fr_iterations,lr_iterations,rank,"
          "compression_ratio,oversampling_ratio,phi_diff_two_norm,psi_diff_two_norm,"
          "fr_converged,lr_converged,speedup,fr_solve_seconds,lr_solve_seconds,"
          "assembly_seconds\n";
    for (const RunResult& r : results) {
      const char* mode = r.has_full && r.has_low ? "both" : (r.has_full ? "full" : "lowrank");
      const ProblemConfig& c = r.config.cfg;
      os << r.run_id << "," << (c.preset.empty() ? "custom" : c.preset) << "," << mode << "," << c.solver.seed << ",";
      os << (r.has_full ? std::to_string(r.full.iterations) : std::string()) << ",";
      os << (r.has_low ? std::to_string(r.low.iterations) : std::string()) << ",";
      if (r.has_low && r.low.has_factors) os << r.low.factors.rank;
      else if (r.has_low && !r.low.history.empty()) os << r.low.history.back().rank;
      os << ",";
      if (r.has_comparison) os << fmt(r.comparison.compression_ratio);
      os << ",";
      if (r.has_low && !r.low.history.empty()) os << fmt(r.low.history.back().oversampling);
      os << ",";
      if (r.has_comparison) os << fmt(r.comparison.phi_diff_two_norm);
      os << ",";
      if (r.has_comparison && r.comparison.has_psi_diff) os << fmt(r.comparison.psi_diff_two_norm);
      os << ",";
      os << (r.has_full ? (r.full.converged ? "1" : "0") : "") << ",";
      os << (r.has_low ? (r.low.converged ? "1" : "0") : "") << ",";
      if (r.has_comparison) os << fmt(r.comparison.speedup);
      os << ",";
      if (r.has_full) os << fmt(r.full.solve_seconds);
      os << ",";
      if (r.has_low) os << fmt(r.low.solve_seconds);
      os << "," << fmt(r.assembly_seconds) << "\n";
    }
  }
  {
    std::ofstream os(out_dir + "/history.csv");
    if (!os) throw std::runtime_error("cannot write history.csv in '" + out_dir + "'");
    os << "run_id,method,iteration,diff_two_norm,diff_inf_norm,rank,oversampling\n";
    for (const RunResult& r : results)
      for (const SolveReport* rep : {r.has_full ? &r.full : nullptr, r.has_low ? &r.low : nullptr}) {
        if (!rep) continue;
        for (size_t i = 0; i < rep->history.size(); ++i) {
          const OuterRecord& h = rep->history[i];
          os << r.run_id << "," << rep->method << "," << (i + 1) << "," << fmt(h.diff_two_norm) << ","
             << fmt(h.diff_inf_norm) << ",";
          if (h.rank >= 0) os << h.rank << "," << fmt(h.oversampling);
          else os << ",";
          os << "\n";
        }
      }
  }
  const bool single = results.size() == 1;
  for (const RunResult& r : results) {
    const std::string suffix = single ? "" : "_" + r.run_id;
    if (r.has_full) {
      write_flux_file(out_dir + "/flux_fr" + suffix + ".txt", r.config.cfg, r.full.phi, false);
      if (log_export) write_flux_file(out_dir + "/flux_fr_log" + suffix + ".txt", r.config.cfg, r.full.phi, true);
    }
    if (r.has_low) {
      write_flux_file(out_dir + "/flux_lr" + suffix + ".txt", r.config.cfg, r.low.phi, false);
      if (log_export) write_flux_file(out_dir + "/flux_lr_log" + suffix + ".txt", r.config.cfg, r.low.phi, true);
    }
  }
}

}  // namespace cuda
}  // namespace rtlr
