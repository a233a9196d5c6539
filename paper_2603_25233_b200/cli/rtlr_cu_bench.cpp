// rtlr_cu_bench: the reference's rtlr_bench driver (proj/tools/rtlr_bench.cpp)
// on the B200 core, through the C ABI only (include/rtlr_cu.h), as a
// reference-side caller would bind it.  Same subcommands, flags, outputs and
// exit codes: 0 success, 2 a driver hit the iteration cap, 3 config error,
// 1 other errors.
//
//   rtlr_cu_bench run   (--preset NAME | --config FILE) [--mode full|lowrank|both]
//                       [--seed S] [--out DIR] [--p P] [--q Q] [--max-iterations N]
//                       [--full-resolution] [--no-dsa] [--log-flux] [--device D]
//   rtlr_cu_bench batch (--preset NAME | --config FILE) --seeds 1,2,3 [same options]
//   rtlr_cu_bench presets
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "rtlr_cu.h"

namespace {

struct Args {
  std::string cmd, preset, config, mode = "both", out = "out";
  long long seed = -1;
  int p = 0, q = 0, max_iterations = 0, device = 0;
  bool full_resolution = false, no_dsa = false, log_flux = false;
  std::vector<long long> seeds;
};

[[noreturn]] void usage(const char* msg) {
  std::fprintf(stderr, "error: %s\nusage: rtlr_cu_bench run|batch|presets [options] (see the source header)\n", msg);
  std::exit(3);
}

Args parse(int argc, char** argv) {
  Args a;
  if (argc < 2) usage("need a subcommand");
  a.cmd = argv[1];
  if (a.cmd != "run" && a.cmd != "batch" && a.cmd != "presets") usage("unknown subcommand");
  for (int i = 2; i < argc; ++i) {
    const std::string k = argv[i];
    auto val = [&]() -> std::string {
      if (i + 1 >= argc) usage(("missing value for " + k).c_str());
      return argv[++i];
    };
    if (k == "--preset") a.preset = val();
    else if (k == "--config") a.config = val();
    else if (k == "--mode") a.mode = val();
    else if (k == "--out") a.out = val();
    else if (k == "--seed" && a.cmd == "run") a.seed = std::atoll(val().c_str());
    else if (k == "--seeds" && a.cmd == "batch") {
      const std::string v = val();
      size_t b = 0;
      while (b <= v.size()) {
        const size_t e = v.find(',', b);
        const std::string t = v.substr(b, e == std::string::npos ? std::string::npos : e - b);
        if (!t.empty()) a.seeds.push_back(std::atoll(t.c_str()));
        if (e == std::string::npos) break;
        b = e + 1;
      }
    } else if (k == "--p") a.p = std::atoi(val().c_str());
    else if (k == "--q") a.q = std::atoi(val().c_str());
    else if (k == "--max-iterations") a.max_iterations = std::atoi(val().c_str());
    else if (k == "--device") a.device = std::atoi(val().c_str());
    else if (k == "--full-resolution") a.full_resolution = true;
    else if (k == "--no-dsa" && a.cmd == "run") a.no_dsa = true;
    else if (k == "--log-flux") a.log_flux = true;
    else usage(("unknown option " + k).c_str());
  }
  return a;
}

int fail(int rc) {
  std::fprintf(stderr, "%s: %s\n", rc == RTLR_CU_CONFIG_ERROR ? "config error" : "error", rtlr_cu_last_error());
  return rc == RTLR_CU_CONFIG_ERROR ? 3 : 1;
}

}  // namespace

int main(int argc, char** argv) {
  const Args a = parse(argc, argv);
  if (a.cmd == "presets") {  // preset_catalog (problem.cpp:202-216) plus the BASELINE configs
    const char* rows[][2] = {
        {"homogeneous(sigma_s,L)", "[-1,1]^2, 16Lx16L cells, CL(8L,4L); constant scattering, Gaussian source"},
        {"variable_scattering", "[-1,1]^2, smooth 0.1..100 scattering ramp; 40x40 CL(16,8), full: 80x80 CL(40,20)"},
        {"pin_cell", "[-1,1]^2, 0.1 inside |x|,|y|<=0.5 else 100; 40x40 CL(16,8), full: 80x80 CL(32,16)"},
        {"lattice", "[0,5]^2 absorber checkerboard, unit source in [2,3]^2; 40x40 CL(16,8), full: 80x80 CL(32,16)"},
        {"C1", "BASELINE: 64x64 [0,1]^2, CL(16,8), sigma_t 1, c 0.9, box source; full-rank check"},
        {"C2", "BASELINE: 128x128, CL(32,16), sigma_t 100, c 0.999, smooth source; low-rank p 4"},
        {"C3", "BASELINE: 256x256 7x7 checkerboard, CL(48,24); low-rank p 8, q 16"},
        {"C4", "BASELINE: 512x512 log-normal random medium, CL(64,32); low-rank p 8, q 16"},
        {"C5", "BASELINE: sweep-throughput grid, sigma_t 1"},
    };
    for (const auto& r : rows) std::printf("%-28s %s\n", r[0], r[1]);
    return 0;
  }
  rtlr_cu_config* cfg = nullptr;
  int rc;
  if (!a.config.empty()) {
    rc = rtlr_cu_config_load(a.config.c_str(), &cfg);
  } else if (!a.preset.empty()) {
    const std::string name = a.full_resolution ? a.preset + ":full" : a.preset;
    rc = rtlr_cu_config_create(name.c_str(), &cfg);
  } else {
    std::fprintf(stderr, "error: need --preset or --config\n");
    return 3;
  }
  if (rc != RTLR_CU_OK) return fail(rc);
  // apply_overrides (rtlr_bench.cpp:20-31)
  if ((rc = rtlr_cu_config_set_mode(cfg, a.mode.c_str())) != RTLR_CU_OK) return fail(rc);
  if (a.seed >= 0 && (rc = rtlr_cu_config_set(cfg, "solver.seed", static_cast<double>(a.seed))) != RTLR_CU_OK)
    return fail(rc);
  if (a.p > 0 && (rc = rtlr_cu_config_set(cfg, "solver.p", a.p)) != RTLR_CU_OK) return fail(rc);
  if (a.q > 0 && (rc = rtlr_cu_config_set(cfg, "solver.q", a.q)) != RTLR_CU_OK) return fail(rc);
  if (a.max_iterations > 0 && (rc = rtlr_cu_config_set(cfg, "solver.max_iterations", a.max_iterations)) != RTLR_CU_OK)
    return fail(rc);
  if (a.no_dsa && (rc = rtlr_cu_config_set(cfg, "solver.use_dsa", 0.0)) != RTLR_CU_OK) return fail(rc);
  if (a.cmd == "batch" && a.seeds.empty()) usage("--seeds is required for batch");
  std::vector<int64_t> seeds(a.seeds.begin(), a.seeds.end());
  std::vector<char> summary(1 << 16);
  int ok = 0;
  rc = rtlr_cu_run(cfg, a.device, seeds.empty() ? nullptr : seeds.data(), static_cast<int>(seeds.size()),
                   a.out.c_str(), a.log_flux ? 1 : 0, summary.data(), summary.size(), &ok);
  rtlr_cu_config_destroy(cfg);
  if (rc != RTLR_CU_OK) return fail(rc);
  std::fputs(summary.data(), stdout);
  std::printf("outputs written to %s\n", a.out.c_str());
  return ok ? 0 : 2;
}
