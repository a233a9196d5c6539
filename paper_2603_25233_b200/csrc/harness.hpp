// Run harness of the reference: the key = value config
// text format (proj/src/problem.cpp:288-459), run / run_assembled with the
// FR-vs-LR comparison (proj/src/report.cpp:60-98) and the metrics / history
// / flux writers (proj/src/report.cpp:101-195), on the GPU solvers.
#pragma once

#include <string>
#include <vector>

#include "problem.hpp"

namespace rtlr {
namespace cuda {

enum class RunMode { Full = 0, LowRank = 1, Both = 2 };  // problem.hpp:83
RunMode run_mode_from_name(const std::string& s);       // problem.cpp:280-285
const char* run_mode_name(RunMode m);

struct RunConfig {
  ProblemConfig cfg;
  RunMode mode = RunMode::Both;
};

// parse_config_text (problem.cpp:329-452): '#' comments, "key = value"
// lines, "preset = name" resets every field it covers (solver parameters
// and run mode are kept), later keys override; ConfigError on unknown keys,
// bad numbers, unknown presets / field kinds and invalid configurations.
RunConfig parse_config_text(const std::string& text);
RunConfig load_config_file(const std::string& path);  // problem.cpp:454-459

struct RunComparison {  // report.hpp:19-31
  double speedup = 0.0, compression_ratio = 0.0, phi_diff_two_norm = 0.0, psi_diff_two_norm = 0.0;
  bool has_psi_diff = false;
};
struct RunResult {  // report.hpp:46-54
  RunConfig config;
  std::string run_id;
  double assembly_seconds = 0.0;
  bool has_full = false, has_low = false, has_comparison = false;
  SolveReport full, low;
  RunComparison comparison;
};

// run_assembled (report.cpp:76-94): solve FR and / or LR as the mode says
// on an assembled problem, compare when both ran (compare_runs,
// report.cpp:60-74; the psi difference on the GPU).  run_config assembles
// first (run, report.cpp:96-99).
RunResult run_assembled(const RunConfig& rc, Problem& P);
RunResult run_config(const RunConfig& rc, int device);
bool all_converged(const RunResult& r);  // report.hpp:52
// rtlr_bench's per-run summary (tools/rtlr_bench.cpp:33-57) and, for
// several low-rank runs, the seed-batch line (:143-165).
std::string run_summary(const RunResult& r);
std::string batch_summary(const std::vector<RunResult>& results);
// write_outputs (report.cpp:118-195): metrics.csv, history.csv and the
// cell-mean flux grids flux_fr / flux_lr (+ _log when log_export; + _<run_id>
// when several results).
void write_outputs(const std::vector<RunResult>& results, const std::string& out_dir, bool log_export);

}  // namespace cuda
}  // namespace rtlr
