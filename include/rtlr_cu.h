/*
 * rtlr_cu.h — C ABI of the B200 (sm_100a) compute core for the rank-adaptive
 * low-rank SI-DSA transport solver of arXiv 2603.25233.
 *
 * The reference (`rtlr`, /root/reference/proj) is a static C++ library whose
 * Eigen-typed functions are its interface; it has no FFI.  Each entry point
 * below is the plain-pointer equivalent of one reference call, cited as
 * file:line.  All functions return an rtlr_cu_status; on failure
 * rtlr_cu_last_error() gives the reference's exception message.  Status
 * codes map 1:1 onto the reference's exception classes:
 *   RTLR_CU_INVALID_ARGUMENT <- std::invalid_argument
 *   RTLR_CU_RUNTIME_ERROR    <- std::runtime_error (e.g. "sweep: singular
 *                               local block", "galerkin_solve: singular
 *                               reduced system", "build_diffusion: ...")
 *   RTLR_CU_CONFIG_ERROR     <- rtlr::ConfigError (problem.hpp:16-18)
 * Non-convergence is not an error (report converged == 0), as in the
 * reference.  One host thread per problem; not reentrant.
 *
 * Vectors use the reference's layout: DOF = (b*nx + a)*4 + my*2 + mx
 * (dg_space.hpp:22,45-46); angular fluxes are column-major N_x x n.
 * `where` selects RTLR_CU_HOST (pageable/pinned host memory; copies are
 * done inside the call) or RTLR_CU_DEVICE (pointers on the problem's GPU).
 */
#ifndef RTLR_CU_H
#define RTLR_CU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  RTLR_CU_OK = 0,
  RTLR_CU_INVALID_ARGUMENT = 1,
  RTLR_CU_RUNTIME_ERROR = 2,
  RTLR_CU_CONFIG_ERROR = 3,
  RTLR_CU_CUDA_ERROR = 4
} rtlr_cu_status;

enum { RTLR_CU_HOST = 0, RTLR_CU_DEVICE = 1 };

typedef struct rtlr_cu_config rtlr_cu_config;   /* ProblemConfig (problem.hpp:69-81) */
typedef struct rtlr_cu_problem rtlr_cu_problem; /* AssembledProblem (problem.hpp:98-106), GPU-resident */
typedef struct rtlr_cu_report rtlr_cu_report;   /* SolveReport (report.hpp:33-44) */

/* ScalarField (dg_space.hpp:10) as a C callback. */
typedef double (*rtlr_cu_field_fn)(void* user, double x, double y);

const char* rtlr_cu_last_error(void);
int rtlr_cu_version(void);
int rtlr_cu_device_count(void);

/* ---- configuration: make_preset (problem.hpp:90, problem.cpp:111-200) plus
 * the BASELINE configs "C1".."C5"; keys as in problem.cpp:372-451
 * ("mesh.nx", "quadrature.n_theta", "solver.eps_si_sa", "solver.p", ...;
 * the short forms "nx", "n_theta", "eps_si_sa", "p" are accepted too) and
 * constant fields "sigma_s_const", "sigma_a_const", "source_const",
 * "boundary_const". */
int rtlr_cu_config_create(const char* preset, rtlr_cu_config** out);
int rtlr_cu_config_set(rtlr_cu_config* cfg, const char* key, double value);
/* which: "sigma_s" | "sigma_a" | "source" | "boundary" */
int rtlr_cu_config_set_field(rtlr_cu_config* cfg, const char* which, rtlr_cu_field_fn fn, void* user);
void rtlr_cu_config_destroy(rtlr_cu_config* cfg);
/* parse_config_text / load_config_file (problem.cpp:329-459): "key = value"
 * lines, '#' comments, "preset = name" resets the fields it covers (solver
 * parameters and run.mode kept), FieldSpec keys "<field>.kind | value |
 * outside | x0 | x1 | y0 | y1 | decay | center_x | center_y" for the
 * reference presets; CONFIG_ERROR with the reference's messages. */
int rtlr_cu_config_parse(const char* text, rtlr_cu_config** out);
int rtlr_cu_config_load(const char* path, rtlr_cu_config** out);
/* run.mode: "full" | "lowrank" | "both" (default both) */
int rtlr_cu_config_set_mode(rtlr_cu_config* cfg, const char* mode);

/* ---- run / run_assembled + write_outputs (report.cpp:60-195), the
 * rtlr_bench driver (tools/rtlr_bench.cpp): assemble once on `device`, solve
 * FR and/or LR per run.mode for the config's seed (nseeds = 0) or for each
 * of `seeds`, compare FR and LR when both ran (psi difference on the GPU),
 * write metrics.csv, history.csv and flux_{fr,lr}[_log][_<run_id>].txt into
 * out_dir (skipped when out_dir is NULL or ""), and the printable summary
 * into summary (NUL-terminated, truncated to summary_cap).  *all_converged
 * = 0 when a driver hit its iteration cap (rtlr_bench exit code 2). */
int rtlr_cu_run(const rtlr_cu_config* cfg, int device, const int64_t* seeds, int nseeds, const char* out_dir,
                int log_flux, char* summary, size_t summary_cap, int* all_converged);

/* ---- assemble_problem (problem.hpp:108, problem.cpp:461-483) + upload.
 * device < 0 assembles on the host only (inputs can be inspected with
 * rtlr_cu_problem_get; GPU entry points then fail with INVALID_ARGUMENT). */
int rtlr_cu_problem_create(const rtlr_cu_config* cfg, int device, rtlr_cu_problem** out);
void rtlr_cu_problem_destroy(rtlr_cu_problem* p);
/* info: nx, ny, n_theta, n_omega_z, n_dofs, n_omega, n_unique_dirs, sigma_t_uniform */
int rtlr_cu_problem_info(const rtlr_cu_problem* p, int64_t info[8]);
/* DG degree K of the problem (DGSpace::degree, dg_space.hpp:38) and its DOFs
 * per cell s = (K+1)^2 (dofs_per_cell, :43).  K != 1 (0, 2..4) problems run
 * rtlr_cu_sweep / rtlr_cu_sweep_async / rtlr_cu_sweep_dirs / rtlr_cu_apply
 * (sweep.cpp:10-57, operators.cpp:283-288 for any K; test_sweep.cpp:142-155);
 * the solvers, rhs_core and the DSA are K = 1 and return INVALID_ARGUMENT. */
int rtlr_cu_problem_degree(const rtlr_cu_problem* p, int* degree, int* dofs_per_cell);
/* Host copies of the assembled inputs: "dirs" (N_Omega x 3), "weights",
 * "source", "sigma_t_blocks" / "sigma_s_blocks" / "sigma_a_blocks"
 * (ncell x s^2, column-major blocks), "sip_bsr" (ncell x 5 x 16: self, west,
 * east, south, north; K = 1), "stream_blocks" (ax-,ax+,ay-,ay+,bx-,bx+,by-,by+,
 * s x s each). */
int rtlr_cu_problem_get(const rtlr_cu_problem* p, const char* what, double* out);
/* Launch work on an external cudaStream_t (NULL: the problem's own stream). */
int rtlr_cu_problem_set_stream(rtlr_cu_problem* p, void* cuda_stream);
/* "pcg_rtol", "pcg_max_iters", "pcg_multigrid" (0: block-Jacobi PCG), "profile_phases"
 * (1: time the low-rank phases, synchronising at their boundaries), "sweep_kernel"
 * (0 auto, 1 skewed wavefront, 2 row scan, 3 row scan on prefactored cell blocks,
 * 4 cluster wavefront for a few directions, 5 direction groups with a fused
 * scalar-flux epilogue: heterogeneous media, one shared right-hand side,
 * 6 the general-degree diagonal wavefront, any K) */
int rtlr_cu_problem_set_option(rtlr_cu_problem* p, const char* key, double value);
int rtlr_cu_synchronize(rtlr_cu_problem* p);

/* ---- sweep(ops, quad, angle, rhs) (sweep.hpp:14-15), batched over n
 * angles: psi[:, k] = (D_{angles[k]} + Sigma_t)^{-1} rhs[:, k] (+ the
 * angle's inflow boundary vector when the problem has one).  rhs_stride = 0
 * shares one right-hand side; angles == NULL means 0..n-1. */
int rtlr_cu_sweep(rtlr_cu_problem* p, const int* angles, int n, const double* rhs,
                  int64_t rhs_stride, double* psi, int64_t psi_stride, int where);
/* Fully asynchronous device variant: d_angles, rhs and psi are device
 * pointers; the launch is enqueued on the problem's stream and the call
 * returns immediately.  A singular local block is reported by the next
 * rtlr_cu_check (which synchronizes the stream). */
int rtlr_cu_sweep_async(rtlr_cu_problem* p, const int* d_angles, int n, const double* d_rhs,
                        int64_t rhs_stride, double* d_psi, int64_t psi_stride);
int rtlr_cu_check(rtlr_cu_problem* p);
/* Same with explicit directions omega_xy[2k], omega_xy[2k+1] (no inflow). */
int rtlr_cu_sweep_dirs(rtlr_cu_problem* p, const double* omega_xy, int n, const double* rhs,
                       int64_t rhs_stride, double* psi, int64_t psi_stride, int where);
/* StreamingOperator::apply (operators.hpp:53-61, operators.cpp:283-288). */
int rtlr_cu_apply(rtlr_cu_problem* p, double omega_x, double omega_y, const double* v, double* out,
                  int where);
/* rhs_core = Sigma_s phi + G (full_rank.cpp:81). */
int rtlr_cu_rhs_core(rtlr_cu_problem* p, const double* phi, double* out, int where);
/* si_step (full_rank.hpp:28-30); psi may be NULL. */
int rtlr_cu_si_step(rtlr_cu_problem* p, const double* phi_prev, double* phi_star, double* psi, int where);
/* DiffusionSystem::solve / correct (diffusion.hpp:16-39); iterations may be NULL. */
int rtlr_cu_dsa_solve(rtlr_cu_problem* p, const double* rhs, double* x, int where, int* iterations);
int rtlr_cu_dsa_correct(rtlr_cu_problem* p, const double* phi_star, const double* phi_prev,
                        double* delta, int where);
/* C5 synthetic sources: rhs[k*n_dofs + i] = U[0,1)(seed, (dir0+k)*n_dofs + i). */
int rtlr_cu_c5_fill(rtlr_cu_problem* p, double* d_rhs, int64_t n_dirs, int64_t dir0, uint64_t seed);

/* ---- drivers */
typedef struct { /* FullRankOptions (full_rank.hpp:32-37) */
  double eps_si_sa;
  int max_iterations;
  int use_dsa;
  int store_psi;
} rtlr_cu_fr_options;

typedef struct { /* LowRankOptions + LowRankParams (low_rank.hpp:29-36, 146-153) */
  int p, q;
  double eps_res, eps_diff, eps_svd, eps_mgs;
  double eps_si_sa;
  int max_iterations;
  int use_dsa;
  uint64_t seed;
  int build_factors;
} rtlr_cu_lr_options;

void rtlr_cu_fr_options_default(rtlr_cu_fr_options* o);
void rtlr_cu_lr_options_default(rtlr_cu_lr_options* o);
/* Options from the problem's SolverParams (report.cpp:20-43 full_options /
 * low_options). */
int rtlr_cu_problem_fr_options(const rtlr_cu_problem* p, rtlr_cu_fr_options* o);
int rtlr_cu_problem_lr_options(const rtlr_cu_problem* p, rtlr_cu_lr_options* o);
/* solve_full_rank (full_rank.hpp:41-43) */
int rtlr_cu_solve_full_rank(rtlr_cu_problem* p, const rtlr_cu_fr_options* o, rtlr_cu_report** out);
/* solve_low_rank (low_rank.hpp:156-158) */
int rtlr_cu_solve_low_rank(rtlr_cu_problem* p, const rtlr_cu_lr_options* o, rtlr_cu_report** out);

/* info: iterations, converged, n_history, has_psi, factor_rank, sampled_total, psi_dofs, n_dofs */
int rtlr_cu_report_info(const rtlr_cu_report* r, int64_t info[8]);
/* "phi", "psi", "S", "X", "V", "solve_seconds", or a per-outer-iteration
 * history column: "diff_two_norm", "diff_inf_norm", "rank", "oversampling",
 * "inner_iterations", "sampled_count", "fullrank_fallback", "dsa_iterations".
 * Low-rank reports also carry "phase_work": 9 x 4 doubles (seconds, algorithmic
 * HBM bytes, flops, calls) for the phases sweep, cgs, projections, galerkin_q,
 * residual_q, build_C, verify, svd, dsa; seconds are -1 unless the problem
 * option "profile_phases" (or RTLR_PROFILE=1) timed them. */
int rtlr_cu_report_get(const rtlr_cu_report* r, const char* what, double* out);
int rtlr_cu_report_sampled(const rtlr_cu_report* r, int* counts, int* flat);
void rtlr_cu_report_destroy(rtlr_cu_report* r);

/* ---- angle sharding for N GPUs (one process per GPU): the angles rank
 * `rank` of `nranks` owns; mirror pairs stay together and quadrants stay
 * balanced.  Pure host logic (no GPU needed). */
int rtlr_cu_partition_angles(int n_theta, int n_omega_z, int nranks, int rank, int* count,
                             int* angles);
/* Low-rank sharding of one phase's list of m angles (sampled sweeps, Galerkin
 * solves, residual norms): rank `rank` owns items [*begin, *end), blocks of
 * *bsz = ceil(m / nranks) items, gathered back in order with one in-place
 * all-gather.  Pure host logic (no GPU needed). */
int rtlr_cu_shard_block(int m, int nranks, int rank, int* begin, int* end, int* bsz);
/* psi_difference (report.cpp:47-58): ||psi_full - X diag(S) V^T||_F with
 * psi_full N_x x N_Omega, X N_x x rank, S rank, V N_Omega x rank (all
 * column-major, e.g. a full-rank report's "psi" and a low-rank report's
 * "X", "S", "V"); the reconstruction is formed 128 angles at a time. */
int rtlr_cu_psi_difference(rtlr_cu_problem* p, const double* psi_full, const double* X, const double* S,
                           const double* V, int rank, double* out, int where);

/* ---- dense kernels of the truncation path, host buffers in and out (for
 * tests and tools): the blocked Householder QR of the low-rank basis rebuild
 * (low_rank.cpp:112-130): a (m x n, m >= n, column-major) = q r, q m x n with
 * orthonormal columns, r n x n upper triangular (Eigen sign conventions). */
int rtlr_cu_dense_qr(int device, int64_t m, int n, const double* a, double* q, double* r);

/* The batched Galerkin solve (low_rank.cpp:176-200) two ways, for tests and
 * tools: m <= 64 systems A_j = omx Px- + omy Py- + Pt (sign-selected among
 * the 5 projections proj[5][r][r], column-major, r = r0 + k) with right-hand
 * side prhs: sol_full by the partial-pivot LU at rank r; sol_border by the
 * rank-r0 factors finished with the k <= 8 border columns (the low-rank
 * loop's prefactored candidates).  Both r x m, column-major. */
int rtlr_cu_dense_galerkin_border(int device, int r0, int k, int m, const int* angles, int n_omega,
                                  const double* dirs, const double* proj, const double* prhs, double* sol_full,
                                  double* sol_border);

/* ---- caller-assembled problems.  The reference's solvers take assembled
 * objects, not a config: solve_full_rank(ops, quad, bc, source, dsa, opts)
 * (full_rank.hpp:41-43), solve_low_rank(...) (low_rank.hpp:156-158),
 * si_step (full_rank.hpp:28-30), sweep (sweep.hpp:14-15), with ops a
 * DiscreteOperators (operators.hpp:17-32), quad an AngularQuadrature
 * (quadrature.hpp:12-20), bc a BoundaryData (full_rank.hpp:11-20) and dsa a
 * DiffusionSystem (diffusion.hpp:16-39).  rtlr_cu_problem_upload takes the
 * same data as plain arrays; every rtlr_cu_problem entry point above then
 * works on it.  K = 1 (4 DOFs per cell, DOF = (b*nx + a)*4 + my*2 + mx); the
 * streaming blocks are those of the mesh (operators.cpp:47-112). */
typedef struct {
  int nx, ny;                      /* SpatialMesh (dg_space.hpp:15-30) */
  double x_min, x_max, y_min, y_max;
  int n_theta, n_omega_z;          /* CL shape of dirs (sharding keeps mirror pairs together); 0, 0: any set */
  int n_omega;
  const double* dirs;              /* n_omega x 3 row-major (Omega_x, Omega_y, Omega_z), quad.dirs */
  const double* weights;           /* n_omega, quad.weights */
  const double* sigma_t_blocks;    /* ncell x 16 (4x4 column-major per cell), ops.sigma_t_blocks */
  const double* sigma_s_blocks;    /* ncell x 16, the blocks of ops.sigma_s */
  const double* sigma_a_blocks;    /* ncell x 16 or NULL (= sigma_t - sigma_s), the blocks of ops.sigma_a */
  const double* source;            /* N_x, the projected source G */
  const double* boundary;          /* n_omega x N_x (bc.per_angle) or NULL: vacuum */
  const double* sip_bsr;           /* ncell x 5 x 16 (self, west, east, south, north) or NULL: built from the blocks */
  int use_dsa;                     /* 0: no diffusion system (dsa == nullptr) */
} rtlr_cu_problem_desc;
int rtlr_cu_problem_upload(const rtlr_cu_problem_desc* desc, int device, rtlr_cu_problem** out);

/* ---- low-rank primitives (low_rank.hpp:18-144), device-resident.  A basis
 * or inner-loop result borrows its problem (as the reference's LowRankBasis
 * borrows ops / quad / bc, low_rank.hpp:89-91): destroy it before the
 * problem. */
typedef struct rtlr_cu_rng rtlr_cu_rng;           /* SubsampleRng (low_rank.hpp:18-27) */
typedef struct rtlr_cu_lr_basis rtlr_cu_lr_basis; /* LowRankBasis (low_rank.hpp:42-102) */
typedef struct rtlr_cu_inner rtlr_cu_inner;       /* InnerLoopResult (low_rank.hpp:125-136) */
typedef struct { /* LowRankParams (low_rank.hpp:29-36) */
  int p, q;
  double eps_res, eps_diff, eps_svd, eps_mgs;
} rtlr_cu_lr_params;
void rtlr_cu_lr_params_default(rtlr_cu_lr_params* o);

/* SubsampleRng: mt19937_64(seed), masked-rejection draw_below (low_rank.cpp:15-27)
 * and the partial Fisher-Yates sample_without_replacement (:29-37);
 * *n_out = min(count, n). */
int rtlr_cu_rng_create(uint64_t seed, rtlr_cu_rng** out);
void rtlr_cu_rng_destroy(rtlr_cu_rng* r);
int rtlr_cu_rng_draw_below(rtlr_cu_rng* r, uint64_t n, uint64_t* out);
int rtlr_cu_rng_sample(rtlr_cu_rng* r, const int* pool, int n, int count, int* out, int* n_out);

/* LowRankBasis(ops, quad, bc, rhs_core) (low_rank.cpp:39-44): an empty
 * basis for this rhs_core (N_x); params carries eps_mgs for
 * mgs_ro_update's overlap trigger and p, q for greedy_subsample. */
int rtlr_cu_lr_basis_create(rtlr_cu_problem* p, const rtlr_cu_lr_params* params, const double* rhs_core, int where,
                            rtlr_cu_lr_basis** out);
void rtlr_cu_lr_basis_destroy(rtlr_cu_lr_basis* b);
/* info: rank, snapshot_count, n_dofs, n_omega */
int rtlr_cu_lr_basis_info(const rtlr_cu_lr_basis* b, int64_t info[4]);
/* "basis" (N_x x rank), "record" (coefficient_record, rank x snapshot_count),
 * "dx_minus" | "dx_plus" | "dy_minus" | "dy_plus" | "sigma_t" (projected_*,
 * rank x rank), "prhs" (X^T rhs_core, rank), "rhs_core" (N_x), all
 * column-major. */
int rtlr_cu_lr_basis_get(const rtlr_cu_lr_basis* b, const char* what, double* out, int where);
int rtlr_cu_lr_basis_sampled(const rtlr_cu_lr_basis* b, int* out); /* sampled_angles(), snapshot_count entries */
/* mgs_ro_update(snapshots, angles, eps_mgs, drop_tol) (low_rank.cpp:66-132);
 * snapshots N_x x n column-major; *reorthogonalized = 1 when the overlap
 * test forced the rebuild. */
int rtlr_cu_lr_mgs_ro_update(rtlr_cu_lr_basis* b, const double* snapshots, const int* angles, int n, double eps_mgs,
                             double drop_tol, int where, int* reorthogonalized);
int rtlr_cu_lr_update_projections(rtlr_cu_lr_basis* b, int reorthogonalized); /* low_rank.cpp:136-174 */
/* galerkin_solve(angle) for m angles (low_rank.cpp:176-200): sol rank x m */
int rtlr_cu_lr_galerkin_solve(rtlr_cu_lr_basis* b, const int* angles, int m, double* sol, int where);
/* residual_norm(angle, c) for m angles (low_rank.cpp:202-215): coeffs rank x m */
int rtlr_cu_lr_residual_norms(rtlr_cu_lr_basis* b, const int* angles, int m, const double* coeffs, double* norms,
                              int where);
/* greedy_subsample(basis, sampled_mask, p, q, rng) (low_rank.cpp:217-252):
 * sampled_mask N_Omega bytes; selected (>= p entries), candidates (>= q),
 * candidate_solutions (rank x q, may be NULL), residual_norms (q, may be
 * NULL); counts in *n_selected, *n_candidates. */
int rtlr_cu_lr_greedy_subsample(rtlr_cu_lr_basis* b, const unsigned char* sampled_mask, int p, int q, rtlr_cu_rng* rng,
                                int* selected, int* n_selected, double* max_residual, int* candidates,
                                int* n_candidates, double* candidate_solutions, double* residual_norms, int where);
/* build_full_coefficients (low_rank.cpp:311-336): C (rank x N_Omega) from the
 * record (sampled angles), m candidate solutions (rank x m, may be m = 0),
 * Galerkin solves for the rest; phi = X (C w) (low_rank.cpp:385). */
int rtlr_cu_lr_build_coefficients(rtlr_cu_lr_basis* b, const int* candidates, int m, const double* candidate_solutions,
                                  double* C, double* phi, int where);
/* truncation_rank (low_rank.cpp:254-266), host arrays */
int rtlr_cu_truncation_rank(const double* s, int n, double eps_svd, int* out);
/* truncate_factors(C, X, eps_svd) (low_rank.cpp:268-277): C rank x N_Omega,
 * X N_x x rank; out X_out (N_x x r'), S_out (r'), V_out (N_Omega x r') with
 * room for r' <= rank; *rank_out = r'.  S_out alone (X_out = V_out = NULL)
 * gives all rank singular values of C (the per-outer-iteration SVD,
 * low_rank.cpp:457). */
int rtlr_cu_truncate_factors(rtlr_cu_problem* p, const double* C, const double* X, int rank, double eps_svd, int where,
                             int* rank_out, double* X_out, double* S_out, double* V_out);
/* low_rank_si(ops, quad, bc, source, phi_prev, params, rng) (low_rank.cpp:340-434) */
int rtlr_cu_low_rank_si(rtlr_cu_problem* p, const double* phi_prev, const rtlr_cu_lr_params* params, rtlr_cu_rng* rng,
                        int where, rtlr_cu_inner** out);
/* info: iterations, rank, sampled_count, reorthogonalizations,
 * verification_rejections, exhausted_all_angles, n_dofs, n_omega */
int rtlr_cu_inner_info(const rtlr_cu_inner* r, int64_t info[8]);
/* "phi_star" (N_x), "coefficients" (rank x N_Omega), "basis" (N_x x rank) */
int rtlr_cu_inner_get(const rtlr_cu_inner* r, const char* what, double* out, int where);
int rtlr_cu_inner_sampled(const rtlr_cu_inner* r, int* out); /* sampled_order, sampled_count entries */
void rtlr_cu_inner_destroy(rtlr_cu_inner* r);

/* NCCL (over NVLink / NVSwitch) for the sharded drivers: rank 0 creates the
 * 128-byte id, the launcher broadcasts it, every rank attaches its problem.
 * solve_full_rank then sweeps this rank's directions and sums the scalar-
 * flux partials with ncclAllReduce (full_rank.cpp:89 psi * w); the DSA
 * correction is replicated.  nranks == 1 with id == NULL detaches. */
int rtlr_cu_nccl_unique_id(unsigned char* id);
int rtlr_cu_problem_set_comm(rtlr_cu_problem* p, int nranks, int rank, const unsigned char* id);

#ifdef __cplusplus
}
#endif

#endif /* RTLR_CU_H */
