// rtlr::cuda — device-resident problem and the solver API that mirrors the
// reference's (proj/include/rtlr/{sweep,full_rank,low_rank,diffusion}.hpp).
#pragma once

#include <algorithm>
#include <chrono>
#include <memory>
#include <iterator>
#include <mutex>
#include <map>
#include <utility>
#include <string>
#include <vector>

#include "device.cuh"
#include "host.hpp"
#include "linalg.cuh"
#include "mg.cuh"
#include "sweep_dgk.cuh"
#include "sweep_het.cuh"

namespace rtlr {
namespace cuda {

// Device (re)allocations made by DBuf (reported with the low-rank profile).
struct AllocStats {
  double seconds = 0.0, bytes = 0.0, free_s = 0.0, malloc_s = 0.0;
  long long count = 0, reused = 0;
  bool split = false;  // RTLR_PROFILE: drain the device first, time the driver calls alone
};
inline AllocStats& alloc_stats() {
  static AllocStats a;
  return a;
}

// A process-wide cache of released DBuf blocks (per device).  The low-rank
// engine's buffers grow with the rank (hundreds of growths per C4 solve):
// cudaFree + cudaMalloc of multi-GB blocks cost 0.05-0.5 s per solve and
// drained the device each time.  Released blocks are kept and handed to the
// next request they fit (at most 4x larger); a reuse drains the device
// first (cudaDeviceSynchronize: the block's previous owner may still have
// work queued on another stream), as the cudaFree it replaces did.  The
// cache holds at most a quarter of the device memory; beyond that the
// largest blocks are freed, and a Problem's destructor frees them all.
class BlockCache {
 public:
  static BlockCache& get() {
    static BlockCache* c = new BlockCache();  // (never destroyed: blocks live until process exit)
    return *c;
  }
  void* take(size_t bytes, size_t* got) {
    std::lock_guard<std::mutex> lk(mu_);
    auto& m = map_[dev()];
    auto it = m.lower_bound(bytes);
    if (it == m.end() || it->first > 4 * bytes) return nullptr;
    void* p = it->second;
    *got = it->first;
    held_[dev()] -= it->first;
    m.erase(it);
    return p;
  }
  // frees every cached block of the current device (a Problem's destructor:
  // the memory goes back to the driver with the problem that used it)
  void trim() {
    std::lock_guard<std::mutex> lk(mu_);
    const int d = dev();
    for (auto& e : map_[d]) cudaFree(e.second);
    map_[d].clear();
    held_[d] = 0;
  }
  void put(void* p, size_t bytes) {
    std::lock_guard<std::mutex> lk(mu_);
    const int d = dev();
    map_[d].emplace(bytes, p);
    held_[d] += bytes;
    if (cap_[d] == 0) {
      size_t fr = 0, tot = 0;
      cudaMemGetInfo(&fr, &tot);
      cap_[d] = tot / 4;
    }
    auto& m = map_[d];
    while (held_[d] > cap_[d] && !m.empty()) {
      auto last = std::prev(m.end());
      cudaFree(last->second);
      held_[d] -= last->first;
      m.erase(last);
    }
  }

 private:
  static int dev() {
    int d = 0;
    cudaGetDevice(&d);
    return d;
  }
  std::mutex mu_;
  std::map<int, std::multimap<size_t, void*>> map_;
  std::map<int, size_t> held_, cap_;
};

template <class T>
class DBuf {
 public:
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { release(); }
  void release() {
    if (p_) BlockCache::get().put(p_, n_ * sizeof(T));
    p_ = nullptr;
    n_ = 0;
  }
  // Grow to at least n elements (contents not preserved).  A buffer that
  // grows again gets 1.5x headroom, so steadily growing work buffers (the
  // low-rank basis raises r every inner iteration) reallocate O(log) times;
  // released blocks are recycled through BlockCache.
  T* ensure(size_t n) {
    if (n > n_) {
      if (alloc_stats().split) cudaDeviceSynchronize();
      const auto t0 = std::chrono::steady_clock::now();
      const size_t want = n_ ? std::max(n, n_ + n_ / 2) : n;
      release();
      const auto t1 = std::chrono::steady_clock::now();
      size_t got = 0;
      void* c = BlockCache::get().take((want ? want : 1) * sizeof(T), &got);
      if (c) {
        RTLR_CUDA(cudaDeviceSynchronize());
        p_ = static_cast<T*>(c);
        n_ = got / sizeof(T);
        ++alloc_stats().reused;
      } else {
        RTLR_CUDA(cudaMalloc(&p_, (want ? want : 1) * sizeof(T)));
        n_ = want;
      }
      alloc_stats().free_s += std::chrono::duration<double>(t1 - t0).count();
      alloc_stats().malloc_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count();
      alloc_stats().seconds += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      alloc_stats().bytes += static_cast<double>(want) * sizeof(T);
      ++alloc_stats().count;
    }
    return p_;
  }
  void upload(const T* h, size_t n, cudaStream_t s) {
    ensure(n);
    if (n) RTLR_CUDA(cudaMemcpyAsync(p_, h, n * sizeof(T), cudaMemcpyHostToDevice, s));
  }
  T* get() const { return p_; }
  size_t size() const { return n_; }
  void swap(DBuf& o) noexcept {
    std::swap(p_, o.p_);
    std::swap(n_, o.n_);
  }

 private:
  T* p_ = nullptr;
  size_t n_ = 0;
};

// proj/include/rtlr/report.hpp:12-50
struct LowRankFactors {
  std::vector<double> X, S, V;  // X: N_x x r, V: N_Omega x r, column-major
  int rank = 0;
};
struct OuterRecord {
  double diff_two_norm = 0.0, diff_inf_norm = 0.0;
  int rank = -1;
  double oversampling = 0.0;
  int inner_iterations = 0, sampled_count = 0;
  bool fullrank_fallback = false;
  int dsa_iterations = 0;  // PCG iterations of this outer step (0: none)
};
struct SolveReport {
  std::string method;
  std::vector<double> phi;
  bool converged = false;
  int iterations = 0;
  double solve_seconds = 0.0;
  long long psi_dofs = 0;
  std::vector<OuterRecord> history;
  bool has_psi = false;
  std::vector<double> psi;  // N_x x N_Omega column-major
  bool has_factors = false;
  LowRankFactors factors;
  std::vector<std::vector<int>> sampled_log;
  // Low-rank phases (lowrank.hpp phase_names order): wall seconds (-1 when
  // not timed), algorithmic HBM bytes, flops, calls.
  std::vector<double> phase_work;  // kPhaseCount x 4
};

struct FullRankOptions {  // full_rank.hpp:32-37
  double eps_si_sa = 1e-6;
  int max_iterations = 500;
  bool use_dsa = true;
  bool store_psi = true;
};
struct LowRankParams {  // low_rank.hpp:29-36
  int p = 1, q = 8;
  double eps_res = 1e-7, eps_diff = 1e-7, eps_svd = 1e-8, eps_mgs = 1e-10;
};
struct LowRankOptions {  // low_rank.hpp:146-153
  LowRankParams inner;
  double eps_si_sa = 1e-6;
  int max_iterations = 500;
  bool use_dsa = true;
  std::uint64_t seed = 0;
  bool build_factors = true;
};

// 128-byte NCCL unique id for a new communicator (rank 0 creates it and
// broadcasts it to the other processes).
void nccl_unique_id(unsigned char* out);

// Assembled problem resident on one GPU.
class Problem {
 public:
  Problem(const ProblemConfig& cfg, int device);
  Problem(HostProblem&& hp, int device);  // caller-assembled (assemble_arrays)
  ~Problem();
  Problem(const Problem&) = delete;
  Problem& operator=(const Problem&) = delete;

  const HostProblem& host() const { return hp_; }
  cudaStream_t stream() const { return stream_; }
  void set_stream(cudaStream_t s);  // external stream (e.g. torch's); nullptr = own

  // Batched sweep, all pointers on the device.  angles may be nullptr
  // (0..n-1 of dirs).  dirs overrides the problem quadrature when given
  // (device pointer, n x 3).
  void sweep(const int* d_angles, int n, const double* d_rhs, long long rhs_stride, double* d_psi,
             long long psi_stride, bool use_bc = true, const double* d_dirs = nullptr);
  // Same with host rhs / psi (pinned for overlap): directions are streamed
  // through device buffers in chunks, H2D / sweep / D2H pipelined on three
  // streams.  h_angles on the host.
  void sweep_host(const int* h_angles, int n, const double* h_rhs, long long rhs_stride, double* h_psi,
                  long long psi_stride);
  // Heterogeneous medium, many directions, one shared right-hand side
  // (the full-rank SI sweeps): the direction-group kernel (sweep_het.cu).
  // weights (per listed angle) and d_phi: the scalar flux sum_k w_k psi_k is
  // formed in the sweep's epilogue (no psi traffic); d_psi (optional) gets
  // column k of angle k (psi_stride).  false when the kernel does not apply
  // (uniform medium, too few directions): nothing was done.
  bool sweep_het(const std::vector<int>& angles, const std::vector<double>* weights, const double* d_rhs,
                 double* d_psi, long long psi_stride, double* d_phi, bool use_bc = true);
  bool het_applies(int n) const;
  // StreamingOperator::apply (operators.cpp:283-288): out = (Sigma_t + Ox Dx + Oy Dy) v
  void apply(double omx, double omy, const double* d_v, double* d_out);
  // DiffusionSystem::solve / correct (diffusion.cpp:203-213); returns PCG iterations
  int dsa_solve(const double* d_rhs, double* d_x);
  int dsa_correct(const double* d_phi_star, const double* d_phi_prev, double* d_delta);
  // rhs_core = Sigma_s phi + G (full_rank.cpp:81)
  void rhs_core(const double* d_phi, double* d_out);
  // si_step (full_rank.cpp:41-58)
  void si_step(const double* d_phi_prev, double* d_phi_star, double* d_psi_or_null);

  SolveReport solve_full_rank(const FullRankOptions& o);
  SolveReport solve_low_rank(const LowRankOptions& o);
  // psi_difference (report.cpp:47-58): || Psi_full - X diag(S) V^T ||_F,
  // device pointers; angles in blocks of 128 (a DMMA GEMM per block plus a
  // fixed-order squared-difference reduction).
  double psi_difference(const double* d_psi, const double* d_X, const double* d_S, const double* d_V, int rank);

  void check_error();  // throws runtime_error("sweep: singular local block")
  // DG degree K != 1 problems run the sweep and the streaming operator only;
  // the K = 1 entry points throw invalid_argument naming `what`.
  int degree() const { return hp_.degree; }
  void require_k1(const char* what) const;
  void release_buffers();  // (destructor) member buffers and the cached blocks back to the driver

  // Direction sharding over ranks (one process per GPU): this rank sweeps
  // its share of the unique directions and the scalar-flux partials are
  // summed with ncclAllReduce.  nranks == 1 restores the unsharded path.
  void set_comm(int nranks, int rank, const void* nccl_unique_id);
  int nranks() const { return nranks_; }
  int rank() const { return rank_; }
  int device() const { return device_; }
  bool sharded() const { return comm_ != nullptr; }
  // Collectives on the problem stream (no-ops without a communicator):
  // in-place all-gather of count_per_rank doubles per rank; max over ranks.
  void allgather_inplace(double* buf, size_t count_per_rank);
  void allreduce_sum(double* d_buf, size_t n);
  void allreduce_max(int* d_buf, int n);
  // check_error() with the singular-block flag max-reduced over the ranks
  // first, so every rank throws together (no rank left in a collective).
  void check_error_all();

  // Unique 2D transport operators: mirror directions (j1, j2) and
  // (j1, n_z-1-j2) have bitwise-identical (Omega_x, Omega_y).
  const std::vector<int>& unique_rep() const { return uniq_rep_; }
  const std::vector<int>& unique_of() const { return uniq_of_; }

  // DSA PCG stop (relative residual).  The reference solves the DSA system
  // directly; at 1e-10 the correction's error stays below the SI
  // iteration's rounding: parity to the oracle's direct solve, outer and
  // low-rank iteration counts are unchanged at C1-C4 for every stop from
  // 1e-13 to 1e-9 (tools/dsa_rtol_sweep.py), with 15-25% fewer PCG
  // iterations than at 1e-13.
  double pcg_rtol = 1e-10;
  int pcg_max_iters = 20000;
  bool pcg_multigrid = true;  // false: block-Jacobi PCG
  bool profile_phases = false;  // time the low-rank phases (synchronises at phase boundaries)
  int sweep_kernel = 0;  // 0 auto, 1 skewed wavefront (sweep.cu), 2 row scan, 3 row scan on prefactored blocks,
                         // 4 cluster wavefront (few directions), 5 direction-group kernel (sweep_het.cu)

 private:
  friend class LowRankEngine;
  void init();
  void upload();
  void dedupe_directions();
  PcgArgs pcg_args(const double* b, double* x);

  HostProblem hp_;
  int device_ = 0;
  cudaStream_t stream_ = nullptr;
  bool own_stream_ = true;
  StreamDev sc_{};
  DBuf<double> dirs_, weights_, sigma_t_, sigma_s_, source_, bc_, sip_, jac_, kblocks_;
  DBuf<int> err_, angle_idx_;
  DBuf<double> line_, norm_work_, pcg_vec_, pcg_part_, uniq_w_, scratch_, hin_[3], hout_[3], pref_;
  DBuf<int> hang_;
  cudaStream_t copy_in_ = nullptr, copy_out_ = nullptr;
  DBuf<PcgState> pcg_state_;
  std::vector<std::unique_ptr<DBuf<double>>> mg_bufs_;
  MgDevice mg_;
  PcgGraph pcg_graph_;  // after the buffers it references
  PcgState* h_state_ = nullptr;
  double* h_pin_ = nullptr;  // small pinned host scratch
  std::vector<int> uniq_rep_, uniq_of_;
  std::vector<double> uniq_w_host_;
  int nranks_ = 1, rank_ = 0;
  void* comm_ = nullptr;  // ncclComm_t
  // direction-group sweep (sweep_het.cu): skewed Sigma_t (built once), the
  // skewed source, trace lines, scalar-flux partials, the cached slot tables
  DBuf<double> sig_skew_, rhs_skew_, het_line_, het_part_, het_w_;
  DBuf<int> het_i_;
  std::vector<int> het_key_;
  std::vector<double> het_wkey_;
  int het_groups_ = 0;
  DBuf<int> my_idx_;      // this rank's unique-direction representatives
  DBuf<double> my_w_;
  std::vector<int> my_rep_host_;
  std::vector<double> my_w_host_;
  int my_n_ = 0;
};

}  // namespace cuda
}  // namespace rtlr
