// Low-rank SI-DSA driver on the GPU (placeholder until the LR engine lands).
#include "problem.hpp"

namespace rtlr {
namespace cuda {

SolveReport Problem::solve_low_rank(const LowRankOptions&) {
  throw std::runtime_error("solve_low_rank: not implemented yet");
}

}  // namespace cuda
}  // namespace rtlr
