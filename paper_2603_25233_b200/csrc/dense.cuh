// Dense fp64 kernels of the low-rank path (K4-K11): tall-skinny GEMMs with
// deterministic split-K, GEMV/dot/norm reductions, the transposed streaming
// stencils for border extension, batched Galerkin LU solves, Householder
// QR and one-sided Jacobi SVD.  All reductions use fixed partitions and
// fixed summation orders (bitwise reproducible across runs).
#pragma once

#include "device.cuh"

namespace rtlr {
namespace cuda {

// C[M x N] (ldc) = A^T B with A: K x M (lda), B: K x N (ldb), K large.
// work >= splits * M * N doubles.  beta_add: C += result instead of C =.
void gemm_tn(int M, int N, long long K, const double* A, long long lda, const double* B, long long ldb,
             double* C, long long ldc, double* work, size_t work_doubles, cudaStream_t s);
// C[M x N] (ldc) = A B (or C -= A B) with A: M x K (lda, M large), B: K x N (ldb), K small.
void gemm_nn(long long M, int N, int K, const double* A, long long lda, const double* B, long long ldb,
             double* C, long long ldc, cudaStream_t s, bool subtract = false);
size_t gemm_tn_work(int M, int N, long long K);

// out[i] = sum_k A[i, k] x[k] for A: n x k (lda) — accumulating into y (y += A x * alpha)
void gemv_n(long long n, int k, const double* A, long long lda, const double* x, double alpha, double* y,
            cudaStream_t s);

// Deterministic dot products / norms: out = sum a*b (partials then fixed-order sum);
// work >= kDotWork doubles
constexpr int kDotWork = 296;
void dot(long long n, const double* a, const double* b, double* work, double* out, cudaStream_t s);
// out = a . B[:, *d_col] (column picked on the device; *d_col < 0 gives 0)
void dot_indirect(long long n, const double* a, const double* B, long long ldb, const int* d_col, double* work,
                  double* out, cudaStream_t s);
void scale_copy(long long n, const double* x, const double* h, double* y, cudaStream_t s);  // y = x / *h
void axpy_dev(long long n, const double* alpha, double sign, const double* x, double* y, cudaStream_t s);

// Transposed / plain streaming matrices on p columns (border extension):
// W = [Dx^- P, (Dx^-)^T P, Dy^- P, (Dy^-)^T P, Sigma_t P], each N_x x p,
// written at W + k*p*ldw.
void stream_products(const StencilArgs& a, int p, const double* P, long long ldp, double* W, long long ldw,
                     cudaStream_t s, int c0 = 0, int c1 = -1);  // cells [c0, c1) only (c1 < 0: all)

// Batched Galerkin solves (low_rank.cpp:176-200): for each of m angles,
// A_j = omx Px + omy Py + Pt (r x r, from the 5 projections with leading
// dimension ldp), LU with partial pivoting, c_j = A_j^{-1} (prhs + extra_j).
// sol: r x m (ldsol); extra optional r x m (Xt g_j).  flags[j] = 1 if the
// solution is not finite.  work >= m * r * r doubles for r > kSmemLuMax.
constexpr int kSmemLuMax = 96;
// Small batches (m <= 64, the greedy candidates) switch to the blocked path
// above r = 64 (tools/lu_bench, 16 systems: the one-CTA shared-memory LU is
// faster up to r = 40, equal at 64, 13% slower at 80, 30% at 96, 2.2x at
// 160); larger batches switch at 96.
constexpr int kSmemLuMaxSmall = 64, kSmemLuSmallBatch = 64;
// (RTLR_LU_SMEM_SMALL=0: 96 for every batch)
int lu_smem_max(int m);
size_t galerkin_work_doubles(int r, int m);
size_t galerkin_work_per_system(int r);  // the blocked path's workspace per system
void galerkin_batch(int r, int m, const int* angles, const double* dirs, const double* proj, long long ldp,
                    long long proj_stride, const double* prhs, const double* extra, double* sol,
                    long long ldsol, int* flags, double* work, cudaStream_t s);

// The greedy candidates' systems factored one inner iteration ahead (at the
// rank r0 the basis had then, on another stream) and finished by bordering
// once the k <= 16 new basis columns' projections exist (dense.cu).  work:
// m * galerkin_work_per_system(r0) doubles, shared by the two calls.
void galerkin_prefactor(int r, int m, const int* angles, const double* dirs, const double* proj, long long ldp,
                        long long proj_stride, const double* prhs, double* work, cudaStream_t s,
                        cudaEvent_t assembled = nullptr);
void galerkin_factored_solve(int r, int m, const double* work, double* sol, long long ldsol, int* flags,
                             cudaStream_t s);
bool galerkin_border_fits(int r0, int k);
void galerkin_border_solve(int r0, int k, int m, const int* angles, const double* dirs, const double* proj,
                           long long ldp, long long proj_stride, const double* prhs, const double* work, double* sol,
                           long long ldsol, int* flags, cudaStream_t s, const int* sysidx = nullptr, int m_stored = -1);

// Householder QR of an m x n (m >= n) column-major matrix (lda), in place;
// tau (n).  Q formed explicitly into q (m x n).  r (n x n) upper.  Blocked
// (panels of kQrBlock columns, block reflectors through tall GEMMs);
// work >= householder_qr_work(m, n) doubles.
constexpr int kQrBlock = 32;
size_t householder_qr_work(long long m, int n);
void householder_qr(long long m, int n, double* a, long long lda, double* tau, double* q, long long ldq,
                    double* r, double* work, size_t work_doubles, cudaStream_t s);

// R only (n x n upper, into r) of the Householder QR of a (m x n, ld lda,
// overwritten), in one cooperative launch; false if cooperative launches
// are unavailable (or RTLR_QR_COOP=0) and nothing was done.
bool householder_r_coop(long long m, int n, double* a, long long lda, double* r, cudaStream_t s);

// One-sided Jacobi on the columns of w (m x n, ld), accumulating the
// rotations in v (n x n) when given.  Afterwards columns of w are mutually
// orthogonal: w = U diag(s), s = column norms.
// work >= n + 8 doubles; sweeps_used (optional) receives the sweep count.
// CholeskyQR2 of a well-conditioned m x n block in place: X <- Q, R (n x n,
// ld n) with X_in = Q R.  Qbuf: m x n scratch; work >= cholqr2_work_doubles.
// false on a non-positive Cholesky pivot (X untouched).
size_t cholqr2_work_doubles(long long m, int n);
bool cholqr2_inplace(long long m, int n, double* X, long long ldx, double* R, double* Qbuf, double* work,
                     size_t work_doubles, int* d_flag, cudaStream_t s);
// Singular values (descending, device d_sv[n]) of the m x n matrix a
// (m >= n, destroyed): cooperative Golub-Kahan bidiagonalisation and
// bisection on the Golub-Kahan tridiagonal.  false: not applicable (no
// cooperative launch, m > 8192, RTLR_SVD=jacobi), nothing launched.
size_t bidiag_work_doubles(long long m, int n);
bool bidiag_singular_values(long long m, int n, double* a, long long lda, double* d_sv, double* work,
                            size_t work_doubles, cudaStream_t s);
void jacobi_svd(long long m, int n, double* w, long long ldw, double* v, int max_sweeps, int* host_rotated,
                double* work, cudaStream_t s, int* sweeps_used = nullptr);

}  // namespace cuda
}  // namespace rtlr
