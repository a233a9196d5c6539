// The low-rank machinery on one GPU: LowRankBasis (low_rank.hpp:42-102),
// greedy_subsample (:114-116), the inner loop low_rank_si (:141-144) and the
// truncation (:120-123), as one device-resident engine.  The C ABI exports
// each reference primitive over it (include/rtlr_cu.h, "low-rank
// primitives"); Problem::solve_low_rank drives it.  Host code only here; the
// kernels are in lowrank.cu / dense.cu.
#pragma once

#include <chrono>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "dense.cuh"
#include "problem.hpp"

namespace rtlr {
namespace cuda {

// Index uploads without stream synchronisation: a ring of pinned host
// staging buffers and device buffers.  Upload j records an event that
// follows all work enqueued before it; reusing slot j % kSlots first waits
// for the event of upload j - kSlots/2, which follows every consumer of the
// slot's previous upload (an upload's consumers are enqueued before the
// next-but-one upload) and its H2D copy.
struct IntRing {
  static constexpr int kSlots = 64;
  struct Slot {
    int* h = nullptr;
    size_t hcap = 0;
    DBuf<int> d;
  };
  Slot slot[kSlots];
  cudaEvent_t ev[kSlots] = {};
  long long count = 0;
  cudaStream_t s = nullptr;
  void init(cudaStream_t st) {
    s = st;
    for (auto& e : ev) RTLR_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  ~IntRing() {
    for (auto& sl : slot)
      if (sl.h) cudaFreeHost(sl.h);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
  }
  int* upload(const std::vector<int>& a) {
    const long long j = count++;
    const int k = static_cast<int>(j % kSlots);
    if (j >= kSlots) RTLR_CUDA(cudaEventSynchronize(ev[(j - kSlots / 2) % kSlots]));
    RTLR_CUDA(cudaEventRecord(ev[k], s));
    Slot& sl = slot[k];
    const size_t n = std::max<size_t>(a.size(), 1);
    if (sl.hcap < n) {
      if (sl.h) RTLR_CUDA(cudaFreeHost(sl.h));
      sl.hcap = std::max<size_t>(n, 4096);
      RTLR_CUDA(cudaMallocHost(&sl.h, sl.hcap * sizeof(int)));
    }
    int* d = sl.d.ensure(n);
    if (!a.empty()) {
      std::memcpy(sl.h, a.data(), a.size() * sizeof(int));
      RTLR_CUDA(cudaMemcpyAsync(d, sl.h, a.size() * sizeof(int), cudaMemcpyHostToDevice, s));
    }
    return d;
  }
};

// Device matrix with geometric growth of its column capacity.
struct DMat {
  DBuf<double> buf;
  long long ld = 0;
  int cap = 0;
  void reserve(long long rows, int cols, cudaStream_t s) {
    if (cols <= cap && rows == ld) return;
    const int nc = std::max({cols, 2 * cap, 16});
    DBuf<double> nb;
    nb.ensure(static_cast<size_t>(rows) * nc);
    if (cap > 0 && rows == ld)
      RTLR_CUDA(cudaMemcpyAsync(nb.get(), buf.get(), static_cast<size_t>(ld) * cap * sizeof(double),
                                cudaMemcpyDeviceToDevice, s));
    RTLR_CUDA(cudaStreamSynchronize(s));
    buf.swap(nb);
    ld = rows;
    cap = nc;
  }
  double* col(int j) const { return buf.get() + static_cast<size_t>(ld) * j; }
};

// Per-phase accounting.  Algorithmic work (bytes that must cross HBM and
// flops, from the shapes of each call: DESIGN.md "Per-phase roofline") is
// always counted (host arithmetic only); wall time per phase needs
// synchronisation at the phase boundaries, so it is taken only with
// RTLR_PROFILE=1 or the problem option "profile_phases".
constexpr int kPhaseCount = 9;
inline const char* const* phase_names() {
  static const char* const names[kPhaseCount] = {"sweep", "cgs", "projections", "galerkin_q", "residual_q",
                                                 "build_C", "verify", "svd", "dsa"};
  return names;
}
struct PhaseTimer {
  bool on = false;
  cudaStream_t s = nullptr;
  std::vector<std::pair<std::string, double>> acc;
  std::chrono::steady_clock::time_point t0;
  std::string cur;
  int idx = -1;  // current phase (always tracked, for the work counters)
  double bytes[kPhaseCount] = {}, flops[kPhaseCount] = {};
  long long calls[kPhaseCount] = {};
  void start(const char* name) {
    idx = -1;
    for (int k = 0; k < kPhaseCount; ++k)
      if (std::string(phase_names()[k]) == name) idx = k;
    if (idx >= 0) ++calls[idx];
    cur = name;
    if (!on) return;
    RTLR_CUDA(cudaStreamSynchronize(s));
    t0 = std::chrono::steady_clock::now();
  }
  void stop() {
    if (on) {
      RTLR_CUDA(cudaStreamSynchronize(s));
      const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      bool found = false;
      for (auto& e : acc)
        if (e.first == cur) {
          e.second += dt;
          found = true;
        }
      if (!found) acc.push_back({cur, dt});
    }
    idx = -1;
  }
  void work(double b, double f) {
    if (idx < 0) return;
    bytes[idx] += b;
    flops[idx] += f;
  }
  double seconds(int k) const {
    for (auto& e : acc)
      if (e.first == phase_names()[k]) return e.second;
    return on ? 0.0 : -1.0;
  }
};

// InnerLoopResult (low_rank.hpp:125-136); phi_star, C and X stay on the
// engine (phi(), C(), X()).
struct InnerResult {
  int iterations = 0, rank = 0, sampled_count = 0, reorthogonalizations = 0, verification_rejections = 0;
  bool exhausted = false;
  std::vector<int> sampled_order;
};

// SubsampleOutcome (low_rank.hpp:104-110); the candidate solutions are the
// engine's device block cand_sol() (rank x candidates.size()).
struct GreedyOutcome {
  std::vector<int> selected;
  double max_residual = 0.0;
  std::vector<int> candidates;
  std::vector<double> residual_norms;
};

// The inner-loop machinery (LowRankBasis + low_rank_si) on one GPU.
class LowRankEngine {
 public:
  LowRankEngine(Problem& P, const LowRankParams& prm);
  ~LowRankEngine();
  LowRankEngine(const LowRankEngine&) = delete;
  LowRankEngine& operator=(const LowRankEngine&) = delete;

  PhaseTimer pt_;
  int reorth_count_ = 0;        // Householder rebuilds (all inner loops)
  int svd_sweeps_ = 0, svd_calls_ = 0;
  long long gal_calls_ = 0, gal_systems_ = 0;
  long long verify_calls_ = 0, verify_angles_ = 0;
  double pf_check_worst_ = 0.0;  // RTLR_LU_PREFACTOR=check
  long long pf_used_ = 0, pf_missed_ = 0;  // prefactored candidate batches finished by bordering / redone in full
  double reorth_seconds_ = 0.0;  // their wall time (meaningful with RTLR_PROFILE=1)
  double cgs_split_[4] = {0, 0, 0, 0};  // RTLR_PROFILE: block GEMMs + host / per-snapshot loop / overlap / GEMMs only
  void lap(int slot, std::chrono::steady_clock::time_point& t) {
    if (!pt_.on) return;
    RTLR_CUDA(cudaStreamSynchronize(s_));
    const auto now = std::chrono::steady_clock::now();
    cgs_split_[slot] += std::chrono::duration<double>(now - t).count();
    t = now;
  }

  // low_rank_si (low_rank.cpp:340-434): the whole inner loop from phi_prev.
  InnerResult inner(const double* d_phi_prev, SubsampleRng& rng);

  // ---- LowRankBasis (low_rank.hpp:42-102), device pointers throughout
  // A fresh, empty basis for rhs_core = Sigma_s phi_prev + G (the
  // reference's constructor argument; low_rank.cpp:349-351 / :39-44).
  void reset(const double* d_phi_prev);
  void reset_rhs(const double* d_rhs_core);
  // mgs_ro_update(snapshots, angles, eps_mgs, drop_tol) (low_rank.cpp:66-132):
  // snaps N_x x angles.size() (ld N_x); true when the overlap test forced
  // the Householder rebuild.
  bool mgs_ro_update(const double* snaps, const std::vector<int>& angles);
  void update_projections(bool reorth);  // low_rank.cpp:136-174
  // galerkin_solve for each listed angle (low_rank.cpp:192-200): d_sol r x m (ldsol)
  void galerkin(const std::vector<int>& angles, double* d_sol, long long ldsol);
  // residual_norm(angle, c) per listed angle (low_rank.cpp:202-208, 283-307)
  std::vector<double> residual_norms(const std::vector<int>& angles, const double* coeffs, long long ldc,
                                     bool mirror_equal = false);
  // greedy_subsample(basis, sampled_mask, p, q, rng) (low_rank.cpp:217-252)
  GreedyOutcome greedy_subsample(const std::vector<char>& sampled, int p, int q, SubsampleRng& rng);
  // build_full_coefficients (low_rank.cpp:311-336) into C(): the record's
  // columns for sampled angles, the given candidate solutions, Galerkin
  // solves for the rest
  void build_full_coefficients(const std::vector<int>* cand, const double* cand_sol);
  void phi_from_C();  // phi = X (C w) (low_rank.cpp:385,394)
  // Thin SVD of C (r x N_Omega): singular values (non-increasing); with U,
  // V the factors X_out = X U[:, :r'] and V[:, :r'] of truncate_factors.
  std::vector<double> svd(bool vectors, int keep, std::vector<double>* Xout, std::vector<double>* Vout);
  // Loads an external coefficient matrix C (r x N_Omega, ld r) and basis
  // X (N_x x r, ld N_x) for svd() / truncate_factors on caller data.
  void load_factors(const double* d_C, const double* d_X, int r);
  void set_drop_tol(double t) { drop_tol_ = t; }
  // Synchronizes and raises a deferred error flag (a singular sweep block
  // or a non-finite Galerkin solution) as the reference's exception.
  void check() {
    flags_enqueue();
    RTLR_CUDA(cudaStreamSynchronize(s_));
    flags_check();
  }
  void set_eps_mgs(double e) { prm_.eps_mgs = e; }

  int rank() const { return rank_; }
  int snapshot_count() const { return n_snap_; }
  const std::vector<int>& sampled() const { return sampled_; }
  const double* X() const { return X_.col(0); }
  long long ldx() const { return X_.ld; }
  const double* record() const { return rec_.get(); }
  long long ldr() const { return ldr_; }
  // projected matrices: 0 Dx-, 1 Dx+, 2 Dy-, 3 Dy+, 4 Sigma_t (ld ldp())
  const double* proj(int k) const { return proj_.get() + static_cast<size_t>(k) * ldp_ * ldp_; }
  long long ldp() const { return ldp_; }
  const double* prhs() const { return prhs_.get(); }
  const double* rhs_core() const { return rhs_core_.get(); }
  const double* C() const { return C_.get(); }
  const double* cand_sol() const { return cand_.get(); }
  double* phi() { return phi_.get(); }
  cudaStream_t stream() const { return s_; }
  long long n() const { return n_; }
  int n_omega() const { return nomega_; }

 private:
  void galerkin_solve(const std::vector<int>& angles, double* d_sol, long long ldsol);
  void grow(int rank_need, int snaps_need);
  // Row slicing of the tall contractions: with a
  // communicator each rank forms X^T B over its cell range and one
  // allreduce sums the M x N block (the CGS projections and the border
  // extension's X^T W); S -= X C runs on the rank's rows and the rows are
  // all-gathered.  RTLR_ROWSLICE_VIRTUAL=R on one GPU runs the same slices
  // one after another and sums them in slice order (the slicing arithmetic
  // without the collective, for tests).
  void tn_rows(int M, int N, const double* A, long long lda, const double* B, long long ldb, double* C, long long ldc);
  void nn_rows_sub(int p, int r, const double* Xm, long long ldx, const double* Cc, long long ldc, double* S,
                   long long lds, bool share);
  long long slice_row(int k) const { return 4LL * slice_c_[k]; }
  int nslice_ = 1, my_slice_ = 0;
  bool vslice_ = false;
  std::vector<int> slice_c_;
  double host_dot(const double* a, const double* b, long long n);
  int* upload_ints(DBuf<int>& buf, const std::vector<int>& a);
  void flags_enqueue();
  void flags_check();
  double* work(size_t need) { return work_.ensure(std::max<size_t>(need, 4096)); }
  // C = A^T B (K = N_x) with its split-K workspace
  void tn(int M, int N, const double* A, long long lda, const double* B, long long ldb, double* C, long long ldc) {
    double* w = work(gemm_tn_work(M, N, n_));
    gemm_tn(M, N, n_, A, lda, B, ldb, C, ldc, w, work_.size(), s_);
  }
  // Angle sharding of one phase's m items over the communicator's ranks
  // (the whole list without one); padded(m) = items incl. the all-gather pad.
  ShardBlock blk(int m) const {
    if (!P_.sharded()) return ShardBlock{0, m, m};
    return shard_block(m, P_.nranks(), P_.rank());
  }
  int padded(int m) const { return P_.sharded() ? blk(m).bsz * P_.nranks() : m; }

  Problem& P_;
  LowRankParams prm_;
  const HostProblem& hp_;
  cudaStream_t s_;
  long long n_;
  int nomega_, rmax_;
  long long ldp_;
  StencilArgs sa_;
  const double* dirs_;
  double drop_tol_ = 1e-12;  // low_rank.hpp:61-62 default
  DMat X_;
  DBuf<double> proj_, prhs_, rhs_core_, phi_, phi_old_, rem_, vec_, C_, work_, snaps_, wbuf_, gbuf_, sol_, cand_,
      ybuf_, nrm_, qa_, qq_, qr_, tau_, hrec_, luw_, gsol_, cgs_, svq_, svr_, svm_, rcoef_;
  DBuf<int> ang_, ang2_, flags_, pos_, rfrom_;
  DBuf<double> tpart_, gath_, npart_;
  double* hbuf_ = nullptr;
  double* hnorm_ = nullptr;  // pinned: residual norms read back per greedy step / verification pass
  size_t hnorm_cap_ = 0;
  void* hstate_ = nullptr;  // pinned CgsState read back once per CGS batch
  int* hflags_ = nullptr;   // pinned: [0] Galerkin non-finite, [1] sweep singular block
  DBuf<int> gal_bad_, chol_flag_;
  IntRing ring_;
  int rank_ = 0, n_snap_ = 0, prev_rank_ = 0;
  // The greedy candidates one inner iteration ahead (lowrank.cu predraw):
  // drawn as soon as the next batch of angles is fixed (the pool and the
  // RNG state are then what greedy_subsample will see), their systems
  // factored at the current rank on s2_ while the next sweep, CGS and
  // projection update run, finished by bordering (dense.cu).
  struct Prefactor {
    bool have_cands = false, factored = false;
    int r0 = 0;
    std::vector<int> cands, reps, pos;
  } pf_;
  bool prefactor_on_ = true;
  cudaStream_t s2_ = nullptr;
  cudaEvent_t ev_fork_ = nullptr, ev_asm_ = nullptr, ev_done_ = nullptr;
  DBuf<double> pfw_;
  DBuf<int> pf_ang_;
  int* pf_hang_ = nullptr;  // pinned staging of the distinct candidates
  void predraw(const std::vector<char>& sampled, const std::vector<int>& next, int q, SubsampleRng& rng);
  GreedyOutcome greedy_evaluate(std::vector<int> cands, int p, bool use_prefactor);
  DBuf<double> rec_;  // coefficient record, rmax x N_Omega (ld ldr_), device-resident
  long long ldr_ = 0;
  int rec_cols_ = 0;
  double* rec_col(int j) { return rec_.get() + static_cast<long long>(j) * ldr_; }
  std::vector<int> sampled_;
};

}  // namespace cuda
}  // namespace rtlr
