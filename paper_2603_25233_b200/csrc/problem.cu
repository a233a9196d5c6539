// rtlr::cuda::Problem: upload, batched sweeps, DSA and the full-rank SI-DSA
// driver (proj/src/full_rank.cpp:41-122) on one B200.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>

#include <nccl.h>

#include "problem.hpp"

namespace rtlr {
namespace cuda {

#define RTLR_NCCL(call)                                                                        \
  do {                                                                                         \
    ncclResult_t r_ = (call);                                                                  \
    if (r_ != ncclSuccess)                                                                     \
      throw ::rtlr::cuda::CudaError(std::string("NCCL error ") + ncclGetErrorString(r_) + " at " + \
                                    __FILE__ + ":" + std::to_string(__LINE__));               \
  } while (0)

void nccl_unique_id(unsigned char* out) {
  ncclUniqueId id;
  RTLR_NCCL(ncclGetUniqueId(&id));
  std::memcpy(out, id.internal, NCCL_UNIQUE_ID_BYTES);
}

void Problem::set_comm(int nranks, int rank, const void* id) {
  if (nranks < 1 || rank < 0 || rank >= nranks) throw std::invalid_argument("set_comm: bad rank layout");
  if (comm_) {
    ncclCommDestroy(static_cast<ncclComm_t>(comm_));
    comm_ = nullptr;
  }
  nranks_ = nranks;
  rank_ = rank;
  if (nranks > 1 || id != nullptr) {
    if (id == nullptr) throw std::invalid_argument("set_comm: nranks > 1 needs an NCCL unique id");
    ncclUniqueId uid;
    std::memcpy(uid.internal, id, NCCL_UNIQUE_ID_BYTES);
    ncclComm_t c;
    RTLR_CUDA(cudaSetDevice(device_));
    RTLR_NCCL(ncclCommInitRank(&c, nranks, uid, rank));
    comm_ = c;
  }
  // this rank's unique directions (mirror pairs never split, so the unique
  // representatives of the owned angles are exactly this rank's share)
  const std::vector<int> mine = partition_angles(hp_.cfg.n_theta, hp_.cfg.n_omega_z, nranks, rank);
  std::vector<char> seen(uniq_rep_.size(), 0);
  std::vector<int> reps;
  std::vector<double> w;
  for (int a : mine) {
    const int u = uniq_of_[a];
    // each distinct operator is swept by the rank owning its representative
    // (CL mirror pairs never split; an arbitrary direction set may)
    if (seen[u] || uniq_rep_[u] != a) continue;
    seen[u] = 1;
    reps.push_back(uniq_rep_[u]);
    w.push_back(uniq_w_host_[u]);
  }
  my_n_ = static_cast<int>(reps.size());
  my_rep_host_ = reps;
  my_w_host_ = w;
  my_idx_.upload(reps.data(), reps.size(), stream_);
  my_w_.upload(w.data(), w.size(), stream_);
  RTLR_CUDA(cudaStreamSynchronize(stream_));
}

namespace {

// 4x4 inverse on the host (block-Jacobi preconditioner), Gauss-Jordan with
// partial pivoting.
void invert4_host(const double* m, double* inv) {
  double a[4][8];
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) {
      a[i][j] = m[j * 4 + i];
      a[i][4 + j] = (i == j) ? 1.0 : 0.0;
    }
  for (int k = 0; k < 4; ++k) {
    int p = k;
    for (int i = k + 1; i < 4; ++i)
      if (std::abs(a[i][k]) > std::abs(a[p][k])) p = i;
    if (a[p][k] == 0.0) throw std::runtime_error("build_diffusion: factorization failed (matrix not positive definite)");
    if (p != k)
      for (int j = 0; j < 8; ++j) std::swap(a[k][j], a[p][j]);
    const double d = a[k][k];
    for (int j = 0; j < 8; ++j) a[k][j] /= d;
    for (int i = 0; i < 4; ++i)
      if (i != k) {
        const double f = a[i][k];
        for (int j = 0; j < 8; ++j) a[i][j] -= f * a[k][j];
      }
  }
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) inv[j * 4 + i] = a[i][4 + j];
}

}  // namespace

Problem::Problem(const ProblemConfig& cfg, int device) : device_(device) {
  assemble(cfg, hp_);
  init();
}

// A caller-assembled problem (rtlr_cu_problem_upload): the host arrays are
// taken as given (assemble_arrays validates and completes them).
Problem::Problem(HostProblem&& hp, int device) : device_(device) {
  hp_ = std::move(hp);
  init();
}

void Problem::init() {
  dedupe_directions();
  if (device_ < 0) return;  // host-only assembly (inspection without a GPU)
  RTLR_CUDA(cudaSetDevice(device_));
  RTLR_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
  own_stream_ = true;
  RTLR_CUDA(cudaMallocHost(&h_state_, sizeof(PcgState)));
  RTLR_CUDA(cudaMallocHost(&h_pin_, 64 * sizeof(double)));
  upload();
}

Problem::~Problem() {
  if (device_ < 0) return;
  cudaSetDevice(device_);
  if (comm_) ncclCommDestroy(static_cast<ncclComm_t>(comm_));
  if (copy_in_) cudaStreamDestroy(copy_in_);
  if (copy_out_) cudaStreamDestroy(copy_out_);
  if (stream_) cudaStreamSynchronize(stream_);
  if (own_stream_ && stream_) cudaStreamDestroy(stream_);
  if (h_state_) cudaFreeHost(h_state_);
  if (h_pin_) cudaFreeHost(h_pin_);
  release_buffers();
}

// The member buffers go back through the block cache (their destructors run
// after this body), so free them here first, then the cached blocks.
void Problem::release_buffers() {
  dirs_.release();
  weights_.release();
  sigma_t_.release();
  sigma_s_.release();
  source_.release();
  bc_.release();
  sip_.release();
  jac_.release();
  kblocks_.release();
  line_.release();
  norm_work_.release();
  pcg_vec_.release();
  pcg_part_.release();
  scratch_.release();
  pref_.release();
  mg_bufs_.clear();
  BlockCache::get().trim();
}

void Problem::set_stream(cudaStream_t s) {
  RTLR_CUDA(cudaStreamSynchronize(stream_));
  if (s == nullptr) {
    if (!own_stream_) {
      RTLR_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
      own_stream_ = true;
    }
    return;
  }
  if (own_stream_) cudaStreamDestroy(stream_);
  stream_ = s;
  own_stream_ = false;
}

void Problem::require_k1(const char* what) const {
  if (hp_.degree != 1)
    throw std::invalid_argument(std::string(what) + ": DG degree K = " + std::to_string(hp_.degree) +
                                " runs the sweep and the streaming operator only on the GPU path (the solvers, "
                                "rhs_core and the DSA are K = 1)");
}

void Problem::upload() {
  const HostProblem& h = hp_;
  cudaStream_t s = stream_;
  if (h.degree != 1) {  // general degree: sweep / apply inputs only
    dirs_.upload(h.dirs.data(), h.dirs.size(), s);
    weights_.upload(h.weights.data(), h.weights.size(), s);
    sigma_t_.upload(h.sigma_t.data(), h.sigma_t.size(), s);
    source_.upload(h.source.data(), h.source.size(), s);
    kblocks_.upload(h.kblocks.data(), h.kblocks.size(), s);
    if (h.bc_any) bc_.upload(h.bc.data(), h.bc.size(), s);
    err_.ensure(1);
    RTLR_CUDA(cudaMemsetAsync(err_.get(), 0, sizeof(int), s));
    RTLR_CUDA(cudaStreamSynchronize(s));
    return;
  }
  std::memcpy(sc_.ax_minus, h.sc.ax_minus, sizeof sc_.ax_minus);
  std::memcpy(sc_.ax_plus, h.sc.ax_plus, sizeof sc_.ax_plus);
  std::memcpy(sc_.ay_minus, h.sc.ay_minus, sizeof sc_.ay_minus);
  std::memcpy(sc_.ay_plus, h.sc.ay_plus, sizeof sc_.ay_plus);
  std::memcpy(sc_.bx_minus, h.sc.bx_minus, sizeof sc_.bx_minus);
  std::memcpy(sc_.bx_plus, h.sc.bx_plus, sizeof sc_.bx_plus);
  std::memcpy(sc_.by_minus, h.sc.by_minus, sizeof sc_.by_minus);
  std::memcpy(sc_.by_plus, h.sc.by_plus, sizeof sc_.by_plus);
  std::memcpy(sc_.trx_r, h.sc.trx_r, sizeof sc_.trx_r);
  std::memcpy(sc_.trx_l, h.sc.trx_l, sizeof sc_.trx_l);
  std::memcpy(sc_.try_r, h.sc.try_r, sizeof sc_.try_r);
  std::memcpy(sc_.try_l, h.sc.try_l, sizeof sc_.try_l);
  dirs_.upload(h.dirs.data(), h.dirs.size(), s);
  weights_.upload(h.weights.data(), h.weights.size(), s);
  sigma_t_.upload(h.sigma_t.data(), h.sigma_t.size(), s);
  sigma_s_.upload(h.sigma_s.data(), h.sigma_s.size(), s);
  source_.upload(h.source.data(), h.source.size(), s);
  if (h.bc_any) bc_.upload(h.bc.data(), h.bc.size(), s);
  err_.ensure(1);
  RTLR_CUDA(cudaMemsetAsync(err_.get(), 0, sizeof(int), s));
  if (!h.sip.empty()) {
    const size_t nc = h.ncell;
    std::vector<double> soa(80 * nc), jac(16 * nc);
    for (size_t c = 0; c < nc; ++c) {
      for (int k = 0; k < 80; ++k) soa[k * nc + c] = h.sip[c * 80 + k];
      double inv[16];
      invert4_host(&h.sip[c * 80], inv);
      for (int e = 0; e < 16; ++e) jac[e * nc + c] = inv[e];
    }
    sip_.upload(soa.data(), soa.size(), s);
    jac_.upload(jac.data(), jac.size(), s);
    pcg_vec_.ensure(7 * static_cast<size_t>(h.ndof));  // r z p q rhs tmp4 x
    // multigrid hierarchy for the preconditioner (mg.cuh)
    std::vector<double> cinv;
    const std::vector<MgLevelHost> lv = build_mg_hierarchy(h.nx, h.ny, h.sip, 64, cinv);
    pcg_graph_.reset();
    mg_bufs_.clear();
    mg_ = MgDevice{};
    mg_.nlev = static_cast<int>(lv.size());
    auto alloc = [&](size_t n) {
      mg_bufs_.push_back(std::make_unique<DBuf<double>>());
      return mg_bufs_.back()->ensure(n);
    };
    for (const MgLevelHost& L : lv) {
      const size_t n = static_cast<size_t>(L.nx) * L.ny;
      mg_.nx.push_back(L.nx);
      mg_.ny.push_back(L.ny);
      double* st = alloc(5 * n);
      RTLR_CUDA(cudaMemcpyAsync(st, L.st.data(), 5 * n * sizeof(double), cudaMemcpyHostToDevice, s));
      mg_.st.push_back(st);
      mg_.x.push_back(alloc(n));
      mg_.b.push_back(alloc(n));
      mg_.t.push_back(alloc(n));
    }
    mg_.ncoarse = lv.back().nx * lv.back().ny;
    mg_.cinv = alloc(cinv.size());
    RTLR_CUDA(cudaMemcpyAsync(mg_.cinv, cinv.data(), cinv.size() * sizeof(double), cudaMemcpyHostToDevice, s));
    RTLR_CUDA(cudaStreamSynchronize(s));
    pcg_part_.ensure(5 * static_cast<size_t>(kNormParts));
    pcg_state_.ensure(1);
  }
  norm_work_.ensure(2 * kNormParts + 8);
  uniq_w_.upload(uniq_w_host_.data(), uniq_w_host_.size(), s);
  angle_idx_.upload(uniq_rep_.data(), uniq_rep_.size(), s);
  RTLR_CUDA(cudaStreamSynchronize(s));
}

void Problem::dedupe_directions() {
  const HostProblem& h = hp_;
  // Mirror-pair deduplication (bitwise-equal Omega_x, Omega_y).
  std::map<std::pair<std::uint64_t, std::uint64_t>, int> seen;
  uniq_rep_.clear();
  uniq_of_.assign(h.n_omega, 0);
  uniq_w_host_.clear();
  for (int j = 0; j < h.n_omega; ++j) {
    std::uint64_t bx, by;
    std::memcpy(&bx, &h.dirs[3 * j], 8);
    std::memcpy(&by, &h.dirs[3 * j + 1], 8);
    auto it = seen.find({bx, by});
    if (it == seen.end()) {
      const int u = static_cast<int>(uniq_rep_.size());
      seen[{bx, by}] = u;
      uniq_rep_.push_back(j);
      uniq_w_host_.push_back(h.weights[j]);
      uniq_of_[j] = u;
    } else {
      uniq_of_[j] = it->second;
      uniq_w_host_[it->second] += h.weights[j];
    }
  }
}

void Problem::check_error() {
  int e = 0;
  RTLR_CUDA(cudaMemcpyAsync(&e, err_.get(), sizeof(int), cudaMemcpyDeviceToHost, stream_));
  RTLR_CUDA(cudaStreamSynchronize(stream_));
  if (e) {
    RTLR_CUDA(cudaMemsetAsync(err_.get(), 0, sizeof(int), stream_));
    throw std::runtime_error("sweep: singular local block");
  }
}

void Problem::check_error_all() {
  allreduce_max(err_.get(), 1);
  check_error();
}

void Problem::allgather_inplace(double* buf, size_t count_per_rank) {
  if (!comm_ || count_per_rank == 0) return;
  RTLR_NCCL(ncclAllGather(buf + static_cast<size_t>(rank_) * count_per_rank, buf, count_per_rank, ncclDouble,
                          static_cast<ncclComm_t>(comm_), stream_));
}

void Problem::allreduce_sum(double* d_buf, size_t n) {
  if (!comm_ || n == 0) return;
  RTLR_NCCL(ncclAllReduce(d_buf, d_buf, n, ncclDouble, ncclSum, static_cast<ncclComm_t>(comm_), stream_));
}

void Problem::allreduce_max(int* d_buf, int n) {
  if (!comm_ || n <= 0) return;
  RTLR_NCCL(ncclAllReduce(d_buf, d_buf, n, ncclInt, ncclMax, static_cast<ncclComm_t>(comm_), stream_));
}

void Problem::sweep(const int* d_angles, int n, const double* d_rhs, long long rhs_stride,
                    double* d_psi, long long psi_stride, bool use_bc, const double* d_dirs) {
  if (n <= 0) return;
  if (hp_.degree != 1 || sweep_kernel == 6) {  // general-degree kernel (sweep_dgk.cu)
    DgkSweepArgs g{};
    g.nx = hp_.nx;
    g.ny = hp_.ny;
    g.n = n;
    g.dirs = d_dirs ? d_dirs : dirs_.get();
    g.angles = d_angles;
    g.rhs = d_rhs;
    g.rhs_stride = rhs_stride;
    g.bc = (use_bc && hp_.bc_any && !d_dirs) ? bc_.get() : nullptr;
    g.bc_stride = hp_.ndof;
    g.psi = d_psi;
    g.psi_stride = psi_stride;
    g.sigma_t = sigma_t_.get();
    if (hp_.degree == 1 && kblocks_.size() == 0) {  // K = 1 through the general kernel (cross-check)
      const double* k1[8] = {hp_.sc.ax_minus, hp_.sc.ax_plus, hp_.sc.ay_minus, hp_.sc.ay_plus,
                             hp_.sc.bx_minus, hp_.sc.bx_plus, hp_.sc.by_minus, hp_.sc.by_plus};
      std::vector<double> kb(8 * 16);
      for (int b = 0; b < 8; ++b) std::copy(k1[b], k1[b] + 16, kb.begin() + 16 * b);
      kblocks_.upload(kb.data(), kb.size(), stream_);
    }
    g.blocks = kblocks_.get();
    g.err = err_.get();
    sweep_dgk(hp_.degree, g, stream_);
    return;
  }
  SweepArgs a{};
  a.nx = hp_.nx;
  a.ny = hp_.ny;
  a.n = n;
  a.dirs = d_dirs ? d_dirs : dirs_.get();
  a.angles = d_angles;
  a.rhs = d_rhs;
  a.rhs_stride = rhs_stride;
  a.bc = (use_bc && hp_.bc_any && !d_dirs) ? bc_.get() : nullptr;
  a.bc_stride = hp_.ndof;
  a.psi = d_psi;
  a.psi_stride = psi_stride;
  a.sigma_t = sigma_t_.get();
  // trace lines (up to 8 warps per direction) or the column-split boundary carries
  a.line = line_.ensure(static_cast<size_t>(n) * 8 * (std::max(hp_.nx, hp_.ny) + 1) * 2);
  a.err = err_.get();
  a.sc = sc_;
  // Kernel choice (option sweep_kernel / RTLR_SWEEP=skew|scan|pref|wave):
  // for a handful of directions (the low-rank solver's p-direction batches,
  // latency-bound) the cluster wavefront, one thread-block cluster per
  // direction, with the cell blocks of a heterogeneous medium inverted ahead
  // of it (launch_sweep_prefactor); otherwise the row-chunk scan kernel in
  // uniform media and the skewed wavefront in heterogeneous ones.
  static const int forced = [] {
    const char* e = std::getenv("RTLR_SWEEP");
    if (!e) return 0;
    const std::string v(e);
    return v == "skew" ? 1 : (v == "scan" ? 2 : (v == "pref" ? 3 : (v == "wave" ? 4 : 0)));
  }();
  static const int wave_cluster = [] {  // RTLR_WAVE_CS: fixed cluster size (tuning)
    const char* e = std::getenv("RTLR_WAVE_CS");
    return e ? std::max(1, std::min(16, std::atoi(e))) : 0;
  }();
  int choice = sweep_kernel ? sweep_kernel : forced;
  int cluster = wave_cluster;
  if (choice == 0 || choice == 4) {
    // a few directions: the cluster wavefront whenever every cluster fits at once
    const int cs = sweep_wave_cluster(a, hp_.sigma_t_uniform);
    if (choice == 0 && cs > 0) choice = 4;
    if (choice == 4 && cluster == 0) cluster = cs > 0 ? cs : 2;
  }
  // Heterogeneous media beyond what the clusters hold at once: the skewed
  // wavefront's single-cell steps beat the row scan's per-cell LU inside the
  // scan (C4: 1024 directions 13.7 vs 22.1 ms, 128: 2.8 vs 4.2 ms; C3: 576
  // directions 2.35 vs 3.1 ms); up to 16 directions the prefactored scan.
  if (choice == 0) choice = hp_.sigma_t_uniform ? 2 : (n <= 16 && hp_.nx % 2 == 0 ? 3 : 1);
  if (choice == 3 && (hp_.sigma_t_uniform || hp_.nx % 2 != 0)) choice = 2;  // nothing to factor / pairs unaligned
  if (choice == 4 && (hp_.nx * 16 * 8 + 8 * 1024 > 220 * 1024)) choice = 2;  // trace lines must fit shared memory
  if (choice == 1) {
    launch_sweep(a, hp_.sigma_t_uniform, stream_);
    return;
  }
  if (choice == 3 || (choice == 4 && !hp_.sigma_t_uniform)) {
    // SoA table, two cells of padding on each side (a lane's cell pair may
    // reach one cell past the row ends; those lanes' values are never used)
    const int planes = choice == 4 ? kPrefMinvDoubles : kPrefDoubles;
    const long long stride = (static_cast<long long>(hp_.ncell) + 5) & ~1LL;
    double* t = pref_.ensure(static_cast<size_t>(n) * planes * stride + 4);
    launch_sweep_prefactor(a, t + 2, stride, stream_, planes);
    a.pref = t + 2;
    a.pref_stride = stride;
  }
  if (choice == 4) {
    launch_sweep_wave(a, hp_.sigma_t_uniform, cluster, stream_);
    return;
  }
  launch_sweep_scan(a, hp_.sigma_t_uniform, stream_);
}

bool Problem::het_applies(int n) const {
  if (sweep_kernel == 5) return !hp_.sigma_t_uniform && n > 0;
  if (sweep_kernel != 0) return false;
  static const bool off = [] {
    const char* e = std::getenv("RTLR_SWEEP");
    return e != nullptr && std::string(e) != "het";
  }();
  return !off && !hp_.sigma_t_uniform && n >= 4 * kHetD;
}

bool Problem::sweep_het(const std::vector<int>& angles, const std::vector<double>* weights, const double* d_rhs,
                        double* d_psi, long long psi_stride, double* d_phi, bool use_bc) {
  if (hp_.degree != 1) return false;
  const int n = static_cast<int>(angles.size());
  if (!het_applies(n)) return false;
  const int nx = hp_.nx, ny = hp_.ny;
  if (!sig_skew_.get()) {  // once per problem: the four skewed copies of Sigma_t
    sig_skew_.ensure(skew_layout_doubles(nx, ny, 8));
    build_skew_layout(nx, ny, sigma_t_.get(), 8, sig_skew_.get(), stream_);
  }
  build_skew_layout(nx, ny, d_rhs, 2, rhs_skew_.ensure(skew_layout_doubles(nx, ny, 2)), stream_);
  // slot tables (cached: the full-rank iteration sweeps the same list every time)
  const bool same = het_key_ == angles && (weights ? het_wkey_ == *weights : het_wkey_.empty());
  if (!same) {
    std::vector<int> orient, slot_angle, slot_pos;
    std::vector<double> slot_w;
    for (int o = 0; o < 4; ++o) {
      std::vector<int> ks;
      for (int k = 0; k < n; ++k) {
        const int j = angles[k];
        const int oj = (hp_.dirs[3 * j] >= 0.0 ? 0 : 1) + (hp_.dirs[3 * j + 1] >= 0.0 ? 0 : 2);  // sweep.cpp:37-38
        if (oj == o) ks.push_back(k);
      }
      for (size_t g0 = 0; g0 < ks.size(); g0 += kHetD) {
        orient.push_back(o);
        for (int d = 0; d < kHetD; ++d) {
          const bool real = g0 + d < ks.size();
          const int k = real ? ks[g0 + d] : -1;
          slot_angle.push_back(real ? angles[k] : -1);
          slot_pos.push_back(k);
          slot_w.push_back(real && weights ? (*weights)[k] : 0.0);
        }
      }
    }
    het_groups_ = static_cast<int>(orient.size());
    std::vector<int> pack(orient);
    pack.insert(pack.end(), slot_angle.begin(), slot_angle.end());
    pack.insert(pack.end(), slot_pos.begin(), slot_pos.end());
    het_i_.ensure(pack.size());
    RTLR_CUDA(cudaMemcpyAsync(het_i_.get(), pack.data(), pack.size() * sizeof(int), cudaMemcpyHostToDevice, stream_));
    het_w_.ensure(slot_w.size());
    RTLR_CUDA(cudaMemcpyAsync(het_w_.get(), slot_w.data(), slot_w.size() * sizeof(double), cudaMemcpyHostToDevice,
                              stream_));
    RTLR_CUDA(cudaStreamSynchronize(stream_));  // the host tables may go
    het_key_ = angles;
    het_wkey_ = weights ? *weights : std::vector<double>();
  }
  const int G = het_groups_;
  SweepHetArgs a{};
  a.nx = nx;
  a.ny = ny;
  a.ngroups = G;
  static const int force_w = [] {  // RTLR_HET_W: warps per direction group (tuning)
    const char* e = std::getenv("RTLR_HET_W");
    return e ? std::atoi(e) : 0;
  }();
  a.W = force_w > 0 ? force_w : sweep_het_warps(nx, ny, G);
  a.ndof = hp_.ndof;
  a.dirs = dirs_.get();
  a.group_orient = het_i_.get();
  a.slot_angle = het_i_.get() + G;
  a.slot_pos = het_i_.get() + G + static_cast<size_t>(G) * kHetD;
  a.slot_weight = d_phi ? het_w_.get() : nullptr;
  a.sig_skew = sig_skew_.get();
  a.rhs_skew = rhs_skew_.get();
  a.bc = (use_bc && hp_.bc_any) ? bc_.get() : nullptr;
  a.bc_stride = hp_.ndof;
  a.psi = d_psi;
  a.psi_stride = psi_stride;
  a.phi_part = d_phi ? het_part_.ensure(static_cast<size_t>(G) * hp_.ndof) : nullptr;
  a.line = het_line_.ensure(static_cast<size_t>(G) * a.W * kHetD * nx * 2);
  a.err = err_.get();
  a.sc = sc_;
  launch_sweep_het(a, stream_);
  if (d_phi) reduce_phi_parts(hp_.ndof, G, a.phi_part, d_phi, stream_);
  return true;
}

void Problem::sweep_host(const int* h_angles, int n, const double* h_rhs, long long rhs_stride, double* h_psi,
                         long long psi_stride) {
  // H2D / sweep / D2H pipelined over direction chunks on three streams with
  // kHostBufs rotating device buffers.  Chunks of ~64 MB keep PCIe at full
  // rate in both directions while the fill and drain of the pipeline stay a
  // small fraction of a call (the sweep of a chunk hides under its copies).
  if (n <= 0) return;
  constexpr int kHostBufs = 3;
  const size_t nd = hp_.ndof;
  if (!copy_in_) RTLR_CUDA(cudaStreamCreateWithFlags(&copy_in_, cudaStreamNonBlocking));
  if (!copy_out_) RTLR_CUDA(cudaStreamCreateWithFlags(&copy_out_, cudaStreamNonBlocking));
  const int chunk = static_cast<int>(std::max<size_t>(1, std::min<size_t>(n, (size_t{64} << 20) / (nd * 8))));
  int* d_ang = hang_.ensure(n);
  RTLR_CUDA(cudaMemcpyAsync(d_ang, h_angles, n * sizeof(int), cudaMemcpyHostToDevice, stream_));
  const bool shared = rhs_stride == 0;
  for (int b = 0; b < kHostBufs; ++b) {
    hin_[b].ensure(shared ? nd : nd * chunk);
    hout_[b].ensure(nd * chunk);
  }
  cudaEvent_t in_done[kHostBufs], comp_done[kHostBufs], out_done[kHostBufs];
  for (int b = 0; b < kHostBufs; ++b) {
    RTLR_CUDA(cudaEventCreateWithFlags(&in_done[b], cudaEventDisableTiming));
    RTLR_CUDA(cudaEventCreateWithFlags(&comp_done[b], cudaEventDisableTiming));
    RTLR_CUDA(cudaEventCreateWithFlags(&out_done[b], cudaEventDisableTiming));
  }
  RTLR_CUDA(cudaStreamSynchronize(stream_));
  if (shared) RTLR_CUDA(cudaMemcpyAsync(hin_[0].get(), h_rhs, nd * 8, cudaMemcpyHostToDevice, copy_in_));
  int k = 0;
  for (int c0 = 0; c0 < n; c0 += chunk, ++k) {
    const int b = k % kHostBufs, c = std::min(chunk, n - c0);
    if (!shared) {
      if (k >= kHostBufs) RTLR_CUDA(cudaStreamWaitEvent(copy_in_, comp_done[b], 0));  // buffer b consumed
      RTLR_CUDA(cudaMemcpy2DAsync(hin_[b].get(), nd * 8, h_rhs + static_cast<size_t>(c0) * rhs_stride,
                                  static_cast<size_t>(rhs_stride) * 8, nd * 8, c, cudaMemcpyHostToDevice, copy_in_));
    }
    RTLR_CUDA(cudaEventRecord(in_done[b], copy_in_));
    RTLR_CUDA(cudaStreamWaitEvent(stream_, in_done[b], 0));
    if (k >= kHostBufs) RTLR_CUDA(cudaStreamWaitEvent(stream_, out_done[b], 0));  // output buffer drained
    sweep(d_ang + c0, c, shared ? hin_[0].get() : hin_[b].get(), shared ? 0 : static_cast<long long>(nd),
          hout_[b].get(), static_cast<long long>(nd));
    RTLR_CUDA(cudaEventRecord(comp_done[b], stream_));
    RTLR_CUDA(cudaStreamWaitEvent(copy_out_, comp_done[b], 0));
    RTLR_CUDA(cudaMemcpy2DAsync(h_psi + static_cast<size_t>(c0) * psi_stride, static_cast<size_t>(psi_stride) * 8,
                                hout_[b].get(), nd * 8, nd * 8, c, cudaMemcpyDeviceToHost, copy_out_));
    RTLR_CUDA(cudaEventRecord(out_done[b], copy_out_));
  }
  RTLR_CUDA(cudaStreamSynchronize(copy_out_));
  RTLR_CUDA(cudaStreamSynchronize(stream_));
  for (int b = 0; b < kHostBufs; ++b) {
    cudaEventDestroy(in_done[b]);
    cudaEventDestroy(comp_done[b]);
    cudaEventDestroy(out_done[b]);
  }
  check_error();
}

void Problem::apply(double omx, double omy, const double* d_v, double* d_out) {
  if (hp_.degree != 1) {
    apply_dgk(hp_.degree, hp_.nx, hp_.ny, sigma_t_.get(), kblocks_.get(), omx, omy, d_v, d_out, stream_);
    return;
  }
  StencilArgs a{hp_.nx, hp_.ny, hp_.ncell, sigma_t_.get(), sc_};
  launch_stream_apply(a, omx, omy, d_v, d_out, stream_);
}

void Problem::rhs_core(const double* d_phi, double* d_out) {
  require_k1("rhs_core");
  sigma_apply(hp_.ndof, sigma_s_.get(), d_phi, nullptr, source_.get(), d_out, stream_);
}

PcgArgs Problem::pcg_args(const double* b, double* x) {
  PcgArgs a{};
  a.nx = hp_.nx;
  a.ny = hp_.ny;
  a.ncell = hp_.ncell;
  a.nparts = kNormParts;
  a.max_iters = pcg_max_iters;
  a.rtol2 = pcg_rtol * pcg_rtol;
  a.sip = sip_.get();
  a.jac = jac_.get();
  a.b = b;
  double* v = pcg_vec_.get();
  const size_t n = hp_.ndof;
  a.x = x ? x : v + 6 * n;
  a.r = v;
  a.z = v + n;
  a.p = v + 2 * n;
  a.q = v + 3 * n;
  double* part = pcg_part_.get();
  a.part_rz = part;
  a.part_pq = part + 2 * kNormParts;
  a.part_rr = part + 3 * kNormParts;
  a.part_bb = part + 4 * kNormParts;
  a.state = pcg_state_.get();
  if (pcg_multigrid) {
    a.mg = &mg_;
    a.tmp4 = v + 5 * n;
  }
  return a;
}

int Problem::dsa_solve(const double* d_rhs, double* d_x) {
  require_k1("dsa_solve");
  if (sip_.get() == nullptr) throw std::invalid_argument("dsa: problem assembled without a diffusion system");
  // the iteration runs on resident vectors (so its captured graph is reused
  // across calls); the solution is copied out
  PcgArgs a = pcg_args(d_rhs, nullptr);
  const int it = pcg_solve(a, h_state_, stream_, &pcg_graph_);
  RTLR_CUDA(cudaMemcpyAsync(d_x, a.x, hp_.ndof * sizeof(double), cudaMemcpyDeviceToDevice, stream_));
  return it;
}

int Problem::dsa_correct(const double* d_phi_star, const double* d_phi_prev, double* d_delta) {
  require_k1("dsa_correct");
  // rhs = Sigma_s (phi* - phi_prev)  (diffusion.cpp:210-213)
  double* rhs = pcg_vec_.get() + 4 * static_cast<size_t>(hp_.ndof);
  sigma_apply(hp_.ndof, sigma_s_.get(), d_phi_star, d_phi_prev, nullptr, rhs, stream_);
  return dsa_solve(rhs, d_delta);
}

void Problem::si_step(const double* d_phi_prev, double* d_phi_star, double* d_psi_or_null) {
  require_k1("si_step");
  const size_t n = hp_.ndof;
  const int nu = static_cast<int>(uniq_rep_.size());
  double* rc = scratch_.ensure(n + n * static_cast<size_t>(nu));
  double* psi_u = rc + n;
  rhs_core(d_phi_prev, rc);
  if (!sweep_het(uniq_rep_, &uniq_w_host_, rc, d_psi_or_null ? psi_u : nullptr, static_cast<long long>(n),
                 d_phi_star)) {
    sweep(angle_idx_.get(), nu, rc, 0, psi_u, static_cast<long long>(n));
    phi_accumulate(static_cast<int>(n), nu, psi_u, static_cast<long long>(n), uniq_w_.get(), d_phi_star, stream_);
  }
  if (d_psi_or_null)
    for (int j = 0; j < hp_.n_omega; ++j)
      RTLR_CUDA(cudaMemcpyAsync(d_psi_or_null + j * n, psi_u + uniq_of_[j] * n, n * sizeof(double),
                                cudaMemcpyDeviceToDevice, stream_));
  check_error();
}

// proj/src/full_rank.cpp:60-122
SolveReport Problem::solve_full_rank(const FullRankOptions& o) {
  require_k1("solve_full_rank");
  if (o.use_dsa && sip_.get() == nullptr)
    throw std::invalid_argument("solve_full_rank: DSA requested but no diffusion system");
  const size_t n = hp_.ndof;
  const int nu = static_cast<int>(uniq_rep_.size());
  SolveReport rep;
  rep.method = "full";
  rep.psi_dofs = static_cast<long long>(n) * hp_.n_omega;
  RTLR_CUDA(cudaStreamSynchronize(stream_));
  const auto t0 = std::chrono::steady_clock::now();

  double* base = scratch_.ensure(5 * n + n * static_cast<size_t>(nu));
  double *phi = base, *phi_star = base + n, *rc = base + 2 * n, *delta = base + 3 * n;
  double* psi_u = base + 5 * n;
  RTLR_CUDA(cudaMemsetAsync(phi, 0, n * sizeof(double), stream_));
  // Direction sharding: with a communicator this rank sweeps only its share
  // of the unique directions and the partial scalar fluxes are summed
  // (ncclAllReduce); everything after (norms, DSA) is replicated.
  const bool sharded = comm_ != nullptr;
  const int nsweep = sharded ? my_n_ : nu;
  const int* sweep_idx = sharded ? my_idx_.get() : angle_idx_.get();
  const double* sweep_w = sharded ? my_w_.get() : uniq_w_.get();
  const std::vector<int>& h_idx = sharded ? my_rep_host_ : uniq_rep_;
  const std::vector<double>& h_w = sharded ? my_w_host_ : uniq_w_host_;
  // Heterogeneous media: the direction-group sweep forms phi* in its
  // epilogue and psi is never written (streaming path, full_rank.cpp:90-97);
  // with store_psi the converged iteration's sweep is repeated once with psi
  // output (bitwise the psi phi* came from).
  const bool het = het_applies(nsweep);
  for (int it = 1; it <= o.max_iterations; ++it) {
    rhs_core(phi, rc);
    if (het) {
      sweep_het(h_idx, &h_w, rc, nullptr, 0, phi_star);
    } else {
      sweep(sweep_idx, nsweep, rc, 0, psi_u, static_cast<long long>(n));
      phi_accumulate(static_cast<int>(n), nsweep, psi_u, static_cast<long long>(n), sweep_w, phi_star, stream_);
    }
    if (sharded)
      RTLR_NCCL(ncclAllReduce(phi_star, phi_star, n, ncclDouble, ncclSum, static_cast<ncclComm_t>(comm_), stream_));
    diff_norms(static_cast<int>(n), phi_star, phi, norm_work_.get(), norm_work_.get() + 2 * kNormParts, stream_);
    RTLR_CUDA(cudaMemcpyAsync(h_pin_, norm_work_.get() + 2 * kNormParts, 2 * sizeof(double),
                              cudaMemcpyDeviceToHost, stream_));
    if (sharded)
      check_error_all();  // synchronizes
    else
      check_error();
    OuterRecord rec;
    rec.diff_two_norm = h_pin_[0];
    rec.diff_inf_norm = h_pin_[1];
    rep.iterations = it;
    if (rec.diff_inf_norm <= o.eps_si_sa) {
      rep.history.push_back(rec);
      rep.converged = true;
      RTLR_CUDA(cudaMemcpyAsync(phi, phi_star, n * sizeof(double), cudaMemcpyDeviceToDevice, stream_));
      break;
    }
    if (o.use_dsa) {
      rec.dsa_iterations = dsa_correct(phi_star, phi, delta);
      vadd(static_cast<int>(n), phi_star, delta, phi, stream_);
    } else {
      RTLR_CUDA(cudaMemcpyAsync(phi, phi_star, n * sizeof(double), cudaMemcpyDeviceToDevice, stream_));
    }
    rep.history.push_back(rec);
  }
  if (!rep.converged)
    RTLR_CUDA(cudaMemcpyAsync(phi, phi_star, n * sizeof(double), cudaMemcpyDeviceToDevice, stream_));
  if (het && o.store_psi && !sharded) {  // psi of the last sweep: its right-hand side is still in rc
    sweep_het(h_idx, &h_w, rc, psi_u, static_cast<long long>(n), nullptr);
    check_error();
  }
  rep.phi.resize(n);
  RTLR_CUDA(cudaMemcpyAsync(rep.phi.data(), phi, n * sizeof(double), cudaMemcpyDeviceToHost, stream_));
  RTLR_CUDA(cudaStreamSynchronize(stream_));
  rep.solve_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (o.store_psi && !sharded) {  // sharded runs keep psi distributed (not gathered)
    rep.has_psi = true;
    rep.psi.resize(n * hp_.n_omega);
    std::vector<double> pu(n * static_cast<size_t>(nu));
    RTLR_CUDA(cudaMemcpyAsync(pu.data(), psi_u, pu.size() * sizeof(double), cudaMemcpyDeviceToHost, stream_));
    RTLR_CUDA(cudaStreamSynchronize(stream_));
    for (int j = 0; j < hp_.n_omega; ++j)
      std::memcpy(&rep.psi[j * n], &pu[uniq_of_[j] * n], n * sizeof(double));
  }
  return rep;
}

}  // namespace cuda
}  // namespace rtlr
